"""World-size-2 multi-process test of the sharded (multi-GPU) host path, on CPU.

Two processes over gloo (127.0.0.1) run exactly the host logic the GPU ranks
run in bench.py / ShardedAssembler.finish: column ranges, the all_gather of the
per-shard counts, offsets, and the point-to-point gather to rank 0 (the
same grouped send/recv the GPU ranks run over NCCL).  The per-rank
column assembly is the oracle's column-subset restatement (the GPU path is
covered by tests/test_gpu_shard.py); rank 0 checks the stitched matrix, the
offsets and the free-column split against the reference's golden fixture.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, tag, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import pyoracle as po
    from paper_1804_05156_b200 import shard
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        g = np.load(os.path.join(ROOT, "tests", "golden", tag + ".npz"))
        d, nodes, elems, flags = int(g["dim"]), g["nodes"], g["elems"], g["flags"]
        n = nodes.shape[0]
        c0, c1 = shard.column_ranges(n, world)[rank]
        sub = po.assemble_columns(d, nodes, elems, np.arange(c0, c1, dtype=np.int32))
        free = g["free_nodes"]
        free_cols = free[(free >= c0) & (free < c1)]
        counts = shard.exchange_counts([c1 - c0, free_cols.size, sub.nnz, 0])
        off = shard.exclusive_offsets(counts)
        info = shard.ShardInfo(rank, world, c0, c1, counts, off)
        import torch
        gathered = shard.gather_csc_to_root(info, torch.from_numpy(np.ascontiguousarray(sub.col_ptr, np.int32)),
                                            torch.from_numpy(np.ascontiguousarray(sub.row_idx, np.int32)),
                                            torch.from_numpy(np.ascontiguousarray(sub.values, np.float64)))
        ok = True
        msg = ""
        # every rank agrees on its global offsets
        ok &= info.nnz_before == int(g["a_col_ptr"][c0])
        ok &= info.free_before == int(np.searchsorted(free, c0))
        ok &= info.nnz_total == int(g["a_col_ptr"][-1])
        if rank == 0:
            cp, ri, va = (t.numpy() for t in gathered)
            ok &= np.array_equal(cp, g["a_col_ptr"])
            ok &= np.array_equal(ri, g["a_row_idx"])
            ok &= va.tobytes() == g["a_values"].tobytes()
            ok &= int(off[-1, 1]) == free.size
            if not ok:
                msg = "stitched matrix differs"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok), msg))
    except Exception as e:  # surface worker failures to the test
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("tag", ["square8_jit", "cube3_mixed_jit", "lshape4"])
def test_sharded_assembly_world2_gloo(tag):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tag, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in out), out
