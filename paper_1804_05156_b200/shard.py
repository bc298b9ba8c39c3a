"""Row-sharded multi-GPU assembly.

One process per GPU.  Every rank holds the mesh (replicated: nodes + elements
are ~1/5 of the output bytes) and owns a contiguous range of CSC columns =
nodes; A is symmetric, so that is also the rank's row block.  Ranks assemble
their columns with no data-path collective (fl_mesh_set_columns restricts the
plan and the column kernel to the range).  The only exchange is one
all_gather of the per-shard counts (n_cols, n_free_cols, nnz, nnz_ff), from
which each rank learns its global offsets: concatenating the shards in rank
order, with col_ptr shifted by the nnz of the ranks before, is bit-for-bit the
reference's single CSC (assembly.hpp:261-300, sparse.hpp:72-110), because every
column is computed from the same items in the same order whichever rank owns
it.  A(free, free) and b_f shard the same way over the free columns.

The host logic here (ranges, offsets, stitching) is device-agnostic and is
covered by world-size-2 gloo tests on CPU (tests/test_shard_gloo.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .api import AssemblyResult, CscMatrix, run
from .context import Context
from .mesh import DeviceMesh, Mesh

COUNT_FIELDS = ("n_cols", "n_free_cols", "nnz", "nnz_ff")


def column_ranges(n_nodes: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous column ranges, rank r gets [c0, c1)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    q, r = divmod(n_nodes, world)
    out, c = [], 0
    for k in range(world):
        n = q + (1 if k < r else 0)
        out.append((c, c + n))
        c += n
    return out


def exclusive_offsets(counts: np.ndarray) -> np.ndarray:
    """counts[world, k] -> offsets[world + 1, k] (row r = sum of ranks < r)."""
    counts = np.asarray(counts, dtype=np.int64)
    off = np.zeros((counts.shape[0] + 1, counts.shape[1]), dtype=np.int64)
    np.cumsum(counts, axis=0, out=off[1:])
    return off


def exchange_counts(local: Sequence[int], device=None, group=None) -> np.ndarray:
    """all_gather of this rank's counts -> [world, len(local)] (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(local), dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return torch.stack(out).cpu().numpy()


@dataclass
class ShardInfo:
    rank: int
    world: int
    col_begin: int
    col_end: int
    counts: np.ndarray   # [world, 4] COUNT_FIELDS of every rank
    offsets: np.ndarray  # [world + 1, 4] exclusive prefix over ranks

    @property
    def nnz_before(self) -> int:
        return int(self.offsets[self.rank, 2])

    @property
    def nnz_ff_before(self) -> int:
        return int(self.offsets[self.rank, 3])

    @property
    def free_before(self) -> int:
        return int(self.offsets[self.rank, 1])

    @property
    def nnz_total(self) -> int:
        return int(self.offsets[-1, 2])


def stitch_csc(m: int, parts: Sequence[tuple[np.ndarray, np.ndarray, np.ndarray]]) -> CscMatrix:
    """Concatenate column shards (local col_ptr from 0, global rows) in rank order."""
    cps, ris, vas = [np.zeros(1, dtype=np.int32)], [], []
    base = 0
    for cp, ri, va in parts:
        cp = np.asarray(cp, dtype=np.int64)
        if cp.size == 0 or cp[0] != 0:
            raise ValueError("shard col_ptr must start at 0")
        cps.append((cp[1:] + base).astype(np.int32))
        ris.append(np.asarray(ri, dtype=np.int32))
        vas.append(np.asarray(va, dtype=np.float64))
        base += int(cp[-1])
    col_ptr = np.concatenate(cps)
    row_idx = np.concatenate(ris) if ris else np.zeros(0, np.int32)
    values = np.concatenate(vas) if vas else np.zeros(0, np.float64)
    return CscMatrix(m, col_ptr.size - 1, col_ptr, row_idx, values)


def gather_csc_to_root(info: "ShardInfo", col_ptr, row_idx, values, root: int = 0, group=None):
    """The verification gather to `root` (SURVEY.md §8(e) collective 2): grouped
    point-to-point sends of every rank's column shard -- col_ptr[1:], row_idx,
    values -- received straight into their slices of the global arrays (NCCL
    send/recv between GPU tensors; gloo moves CPU tensors).  Root then shifts
    each shard's pointers by the nnz of the ranks before it.  Returns the global
    (col_ptr, row_idx, values) tensors on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    off = info.offsets
    cp_l, ri_l, va_l = col_ptr, row_idx, values
    if rank != root:
        ops = []
        if int(info.counts[rank, 0]) > 0:
            ops.append(dist.P2POp(dist.isend, cp_l[1:].contiguous(), root, group))
        if int(info.counts[rank, 2]) > 0:
            ops.append(dist.P2POp(dist.isend, ri_l.contiguous(), root, group))
            ops.append(dist.P2POp(dist.isend, va_l.contiguous(), root, group))
        for req in (dist.batch_isend_irecv(ops) if ops else []):
            req.wait()
        return None
    n, nnz = int(off[-1, 0]), int(off[-1, 2])
    dev = ri_l.device
    cp = torch.zeros(n + 1, dtype=torch.int32, device=dev)
    ri = torch.empty(nnz, dtype=torch.int32, device=dev)
    va = torch.empty(nnz, dtype=torch.float64, device=dev)
    ops = []
    for r in range(world):
        c0, c1, z0, z1 = int(off[r, 0]), int(off[r + 1, 0]), int(off[r, 2]), int(off[r + 1, 2])
        if r == root:
            cp[c0 + 1:c1 + 1] = cp_l[1:]
            ri[z0:z1] = ri_l
            va[z0:z1] = va_l
            continue
        if c1 > c0:
            ops.append(dist.P2POp(dist.irecv, cp[c0 + 1:c1 + 1], r, group))
        if z1 > z0:
            ops.append(dist.P2POp(dist.irecv, ri[z0:z1], r, group))
            ops.append(dist.P2POp(dist.irecv, va[z0:z1], r, group))
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    for r in range(world):
        c0, c1, z0 = int(off[r, 0]), int(off[r + 1, 0]), int(off[r, 2])
        if z0:
            cp[c0 + 1:c1 + 1] += z0
    return cp, ri, va


def gather_to_root(obj, root: int = 0, group=None):
    """Host objects of all ranks on `root` (list in rank order), None elsewhere."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = [None] * world if dist.get_rank(group) == root else None
    dist.gather_object(obj, out, dst=root, group=group)
    return out


class ShardedAssembler:
    """This rank's share of fl_assemble: a device mesh restricted to the rank's
    column range, the asynchronous assembly, and the count exchange."""

    def __init__(self, mesh: Mesh, rank: int, world: int, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.mesh = mesh
        self.rank, self.world = rank, world
        self.col_begin, self.col_end = column_ranges(mesh.num_nodes(), world)[rank]
        self.dm = DeviceMesh(self.ctx, mesh)
        self.dm.set_columns(self.col_begin, self.col_end)

    def assemble(self, what: int, f=None, coef=None, g_dirichlet=None, g_neumann=None,
                 result: Optional[AssemblyResult] = None) -> AssemblyResult:
        return run(self.mesh, what, f=f, coef=coef, g_dirichlet=g_dirichlet,
                   g_neumann=g_neumann, ctx=self.ctx, result=result, device_mesh=self.dm)

    def local_counts(self, res: AssemblyResult) -> list[int]:
        s = res.sizes()
        want_sys = bool(getattr(res, "_what", 0) & _lib.OUT_SYSTEM)
        return [s.n, s.n_free_cols if want_sys else 0, s.nnz, s.nnz_ff if want_sys else 0]

    def finish(self, res: AssemblyResult, device=None, group=None) -> ShardInfo:
        """Synchronise the local assembly and exchange counts across ranks."""
        local = self.local_counts(res)
        if self.world == 1:
            counts = np.asarray([local], dtype=np.int64)
        else:
            counts = exchange_counts(local, device=device, group=group)
        return ShardInfo(self.rank, self.world, self.col_begin, self.col_end, counts,
                         exclusive_offsets(counts))
