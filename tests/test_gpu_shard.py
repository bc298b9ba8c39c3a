"""GPU: the B200 path against the reference's golden fixtures, and the
column-sharded (multi-GPU) path against the unsharded one.

Sharding runs every rank's column range on the one GPU in turn (no rank waits
on another: the ranks are independent by construction); the
stitched shards must equal the reference's single CSC bit for bit, for each
column kernel (FL_KERNEL=0 the default label-space pipeline, 1 general, 2 tiled,
3 register-centric).
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from paper_1804_05156_b200 import _lib
from paper_1804_05156_b200.mesh import Mesh
from paper_1804_05156_b200.shard import ShardedAssembler, column_ranges, exclusive_offsets, stitch_csc
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
IDS = [os.path.basename(p)[:-4] for p in GOLDEN]


def _mesh(g):
    return Mesh(int(g["dim"]), g["nodes"], g["elems"], g["flags"])


def _bits(x):
    return np.asarray(x, dtype=np.float64).tobytes()


@pytest.mark.parametrize("path", GOLDEN, ids=IDS)
def test_gpu_matches_golden(path, ctx):
    g = np.load(path)
    m = _mesh(g)
    a = fl.assemble_blockwise(m, ctx=ctx)
    np.testing.assert_array_equal(a.col_ptr, g["a_col_ptr"])
    np.testing.assert_array_equal(a.row_idx, g["a_row_idx"])
    assert _bits(a.values) == _bits(g["a_values"])
    ac = fl.assemble_blockwise(m, coef=g["coef"], ctx=ctx)
    np.testing.assert_array_equal(ac.col_ptr, g["ac_col_ptr"])
    assert _bits(ac.values) == _bits(g["ac_values"])
    for kind, spec in [(1, 1.0), (3, "x"), (4, "xyz")]:
        assert _bits(fl.assemble_load(m, spec, ctx=ctx)) == _bits(g[f"b_{kind}"]), kind
    p = fl.partition_boundary(m, ctx=ctx)
    np.testing.assert_array_equal(p.dirichlet_nodes, g["dir_nodes"])
    np.testing.assert_array_equal(p.free_nodes, g["free_nodes"])
    if g["dir_nodes"].size:
        s = fl.poisson_system(m, 1.0, "x", ctx=ctx)
        assert _bits(s.u0) == _bits(g["u0_x"])
        assert _bits(s.b_mod) == _bits(g["bmod_x"])
        np.testing.assert_array_equal(s.a_ff.col_ptr, g["aff_col_ptr"])
        np.testing.assert_array_equal(s.a_ff.row_idx, g["aff_row_idx"])
        assert _bits(s.a_ff.values) == _bits(g["aff_values"])
    if np.any(g["flags"] == 2):
        r = fl.run(m, _lib.OUT_LOAD | _lib.OUT_PARTITION, f=1.0, g_neumann=1.5, ctx=ctx)
        assert _bits(r.vector(_lib.B)) == _bits(g["b_neumann_const15"])


def _shards(m, world, what, ctx, **fields):
    out = []
    for r in range(world):
        sa = ShardedAssembler(m, r, world, ctx=ctx)
        res = sa.assemble(what, **fields)
        out.append((sa, res, sa.local_counts(res)))
    return out


@pytest.mark.parametrize("kernel", ["0", "1", "2", "3"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("tag", ["square8_jit", "cube3_mixed_jit", "lshape4_jit"])
def test_sharded_stiffness_and_load(tag, world, kernel, ctx, monkeypatch):
    monkeypatch.setenv("FL_KERNEL", kernel)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", tag + ".npz"))
    m = _mesh(g)
    parts = _shards(m, world, _lib.OUT_STIFFNESS | _lib.OUT_LOAD, ctx, f=1.0)
    full = stitch_csc(m.num_nodes(), [(r.matrix().col_ptr, r.matrix().row_idx, r.matrix().values)
                                      for _, r, _ in parts])
    np.testing.assert_array_equal(full.col_ptr, g["a_col_ptr"])
    np.testing.assert_array_equal(full.row_idx, g["a_row_idx"])
    assert _bits(full.values) == _bits(g["a_values"])
    b = np.concatenate([r.vector(_lib.B) for _, r, _ in parts])
    assert _bits(b) == _bits(g["b_1"])
    off = exclusive_offsets(np.asarray([c for _, _, c in parts]))
    for k, (c0, _) in enumerate(column_ranges(m.num_nodes(), world)):
        assert off[k, 2] == g["a_col_ptr"][c0]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("gspec", [0.0, "x"])
@pytest.mark.parametrize("tag", ["square8_jit", "cube3_mixed_jit"])
def test_sharded_system(tag, gspec, world, ctx):
    """A(free, free), b_f, u0, b_mod split by column range (lift path included)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", tag + ".npz"))
    m = _mesh(g)
    ref = fl.poisson_system(m, 1.0, gspec, ctx=ctx)
    parts = _shards(m, world, _lib.OUT_SYSTEM, ctx, f=1.0, g_dirichlet=gspec)
    aff = stitch_csc(ref.a_ff.m, [(r.matrix_ff().col_ptr, r.matrix_ff().row_idx,
                                   r.matrix_ff().values) for _, r, _ in parts])
    np.testing.assert_array_equal(aff.col_ptr, ref.a_ff.col_ptr)
    np.testing.assert_array_equal(aff.row_idx, ref.a_ff.row_idx)
    assert _bits(aff.values) == _bits(ref.a_ff.values)
    for which, full in [(_lib.U0, ref.u0), (_lib.B_MOD, ref.b_mod), (_lib.B_F, ref.b_f),
                        (_lib.B, ref.b)]:
        got = np.concatenate([r.vector(which) for _, r, _ in parts])
        assert _bits(got) == _bits(full), which
    for _, r, _ in parts:  # the partition outputs stay global
        np.testing.assert_array_equal(r.partition().free_nodes, ref.partition.free_nodes)


@pytest.mark.parametrize("world", [2, 4, 7])
@pytest.mark.parametrize("name,n", [("C5", 12), ("C3", 48)])
def test_sharded_label_pipeline_permuted(name, n, world, ctx, ref_which):
    """Random node ids (the C3 / C5 recipes at small n): every shard's columns are
    scattered over the domain; the label-space pipeline orders the owned nodes
    first.  Stitched A, A(free, free) and vectors against the reference, and the
    asynchronous re-plan (FL_REPLAN) on a range set earlier."""
    from paper_1804_05156_b200 import configs
    cfg = configs.build(name, n=n, f_mode="samples")
    m = cfg.mesh
    coef = configs.host_samples(m, rule=1, kind=7) if cfg.coef else None
    a = po.assemble_blockwise(m.dim, m.nodes, m.elems, coef=coef, which=ref_which)
    ref = fl.poisson_system(m, cfg.f, "x", coef=coef, ctx=ctx)
    fields = dict(f=cfg.f, g_dirichlet="x", coef=coef)
    first, second, keep = [], [], []
    for r in range(world):
        sa = ShardedAssembler(m, r, world, ctx=ctx)
        keep.append(sa)  # the device mesh outlives its results' fl_result_sizes
        first.append(sa.assemble(_lib.OUT_SYSTEM, **fields))
        # the same range again, re-planned asynchronously with the first plan's bounds
        second.append(sa.assemble(_lib.OUT_SYSTEM | _lib.REPLAN, **fields))
    for parts in (first, second):
        full = stitch_csc(m.num_nodes(), [(r.matrix().col_ptr, r.matrix().row_idx, r.matrix().values)
                                          for r in parts])
        np.testing.assert_array_equal(full.col_ptr, a.col_ptr)
        np.testing.assert_array_equal(full.row_idx, a.row_idx)
        assert _bits(full.values) == _bits(a.values)
        aff = stitch_csc(ref.a_ff.m, [(r.matrix_ff().col_ptr, r.matrix_ff().row_idx,
                                       r.matrix_ff().values) for r in parts])
        np.testing.assert_array_equal(aff.col_ptr, ref.a_ff.col_ptr)
        np.testing.assert_array_equal(aff.row_idx, ref.a_ff.row_idx)
        assert _bits(aff.values) == _bits(ref.a_ff.values)
        for which, want in [(_lib.U0, ref.u0), (_lib.B_MOD, ref.b_mod), (_lib.B_F, ref.b_f), (_lib.B, ref.b)]:
            assert _bits(np.concatenate([r.vector(which) for r in parts])) == _bits(want), which


def test_set_columns_rejects_bad_range(ctx):
    g = np.load(GOLDEN[0])
    dm = _mesh(g).device(ctx)
    with pytest.raises(fl.Error):
        dm.set_columns(2, 1)
    with pytest.raises(fl.Error):
        dm.set_columns(0, g["nodes"].shape[0] + 1)


@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("tag", ["square8_jit", "cube3_mixed_jit", "lshape4_jit"])
def test_bucketed_plan_matches_golden(tag, world, ctx, monkeypatch):
    """The bucketed plan (used for large meshes) forced on small ones."""
    monkeypatch.setenv("FL_PLAN", "1")
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", tag + ".npz"))
    m = _mesh(g)
    parts = _shards(m, world, _lib.OUT_STIFFNESS | _lib.OUT_LOAD, ctx, f=1.0)
    full = stitch_csc(m.num_nodes(), [(r.matrix().col_ptr, r.matrix().row_idx, r.matrix().values)
                                      for _, r, _ in parts])
    np.testing.assert_array_equal(full.col_ptr, g["a_col_ptr"])
    np.testing.assert_array_equal(full.row_idx, g["a_row_idx"])
    assert _bits(full.values) == _bits(g["a_values"])
    assert _bits(np.concatenate([r.vector(_lib.B) for _, r, _ in parts])) == _bits(g["b_1"])


def test_async_replan_after_new_connectivity(ctx):
    """fl_mesh_set_elems + FL_REPLAN re-plans asynchronously with the old bounds;
    fl_result_sizes refreshes them (and re-runs the column pass if exceeded)."""
    import ctypes as C
    from paper_1804_05156_b200 import api
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "square8_jit.npz"))
    m = _mesh(g)
    rng = np.random.default_rng(5)
    perm = rng.permutation(m.num_nodes()).astype(np.int32)   # node k -> perm[k]
    inv = np.argsort(perm)
    elems_b = perm[m.elems].astype(np.int32)
    nodes_b = np.ascontiguousarray(m.nodes.reshape(-1, 2)[inv])
    mb = Mesh(2, nodes_b, elems_b, g["flags"])
    want = fl.assemble_blockwise(mb, ctx=ctx)
    L = _lib.lib()
    dm = m.device(ctx)
    dm.plan()
    _lib.check(L.fl_mesh_set_elems(ctx.handle, dm.handle, elems_b.ctypes.data, _lib.MEM_HOST))
    _lib.check(L.fl_mesh_set_nodes(ctx.handle, dm.handle, nodes_b.ctypes.data, _lib.MEM_HOST))
    res = api.run(mb, _lib.OUT_STIFFNESS | _lib.REPLAN, ctx=ctx, device_mesh=dm)
    got = res.matrix()
    np.testing.assert_array_equal(got.col_ptr, want.col_ptr)
    np.testing.assert_array_equal(got.row_idx, want.row_idx)
    assert _bits(got.values) == _bits(want.values)
    # a topology with a higher-valence node than the old bounds allow (fan of 40)
    k = 40
    ang = 2 * np.pi * np.arange(k) / k
    fan_nodes = np.vstack([[0.0, 0.0], np.stack([np.cos(ang), np.sin(ang)], 1)])
    fan_elems = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)], dtype=np.int32)
    small = Mesh(2, fan_nodes, np.array([[1 + i, 1 + (i + 1) % k, 1 + (i + 2) % k]
                                         for i in range(k)], dtype=np.int32))
    from tests.meshes import fix_orientation
    small = Mesh(2, fan_nodes, fix_orientation(2, fan_nodes, small.elems))
    fan = Mesh(2, fan_nodes, fix_orientation(2, fan_nodes, fan_elems))
    want = fl.assemble_blockwise(fan, ctx=ctx)
    dm2 = small.device(ctx)
    dm2.plan()
    fe = np.ascontiguousarray(fan.elems, dtype=np.int32)
    _lib.check(L.fl_mesh_set_elems(ctx.handle, dm2.handle, fe.ctypes.data, _lib.MEM_HOST))
    res = api.run(fan, _lib.OUT_STIFFNESS | _lib.REPLAN, ctx=ctx, device_mesh=dm2)
    got = res.matrix()
    np.testing.assert_array_equal(got.col_ptr, want.col_ptr)
    np.testing.assert_array_equal(got.row_idx, want.row_idx)
    assert _bits(got.values) == _bits(want.values)


def test_replan_valence_class_change(ctx):
    """The label plan's segments hold 8 keys per node while the mesh's valence is
    <= 8 (2-D).  New connectivity with a valence-12 node, re-planned asynchronously:
    the first assembly overflows the segments and is redone on the general kernel,
    the next one plans 16-key segments and stays on the fast kernel -- all bitwise."""
    from tests.meshes import fix_orientation
    k = 12
    ang = 2 * np.pi * np.arange(k) / k
    nodes = np.vstack([[0.0, 0.0], np.stack([np.cos(ang), np.sin(ang)], 1)])
    ring = np.array([[1 + i, 1 + (i + 1) % k, 1 + (i + 2) % k] for i in range(k)], dtype=np.int32)
    fan = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)], dtype=np.int32)
    low = Mesh(2, nodes, fix_orientation(2, nodes, ring))    # valence 3
    high = Mesh(2, nodes, fix_orientation(2, nodes, fan))    # node 0: valence 12
    want = fl.assemble_blockwise(high, ctx=ctx)
    dm = low.device(ctx)
    dm.plan()
    fl.run(low, _lib.OUT_STIFFNESS, ctx=ctx, device_mesh=dm).sizes()
    fe = np.ascontiguousarray(high.elems, dtype=np.int32)
    _lib.check(_lib.lib().fl_mesh_set_elems(ctx.handle, dm.handle, fe.ctypes.data, _lib.MEM_HOST))
    for _ in range(3):
        got = fl.run(high, _lib.OUT_STIFFNESS | _lib.REPLAN, ctx=ctx, device_mesh=dm).matrix()
        np.testing.assert_array_equal(got.col_ptr, want.col_ptr)
        np.testing.assert_array_equal(got.row_idx, want.row_idx)
        assert _bits(got.values) == _bits(want.values)


@pytest.mark.parametrize("overlap", ["0", "1"])
def test_replan_side_stream(overlap, monkeypatch, ref_which):
    """FL_OVERLAP: on a re-plan the partition + FaceLists run on the context's side
    stream beside the label plan (1, default) or on the one stream (0) -- same bits."""
    from paper_1804_05156_b200 import configs
    monkeypatch.setenv("FL_OVERLAP", overlap)
    c2 = fl.Context(0)
    cfg = configs.build("C5", n=10, f_mode="samples")
    m = cfg.mesh
    coef = configs.host_samples(m, rule=1, kind=7)
    a = po.assemble_blockwise(m.dim, m.nodes, m.elems, coef=coef, which=ref_which)
    d, f, _, _ = po.partition_boundary(m.dim, m.nodes, m.elems, m.bd_flags, which=ref_which)
    res = fl.AssemblyResult(c2)
    dm = m.device(c2)
    for what in (_lib.OUT_SYSTEM, _lib.OUT_SYSTEM | _lib.REPLAN, _lib.OUT_SYSTEM | _lib.REPLAN):
        r = fl.run(m, what, f=cfg.f, coef=coef, g_dirichlet="x", ctx=c2, result=res, device_mesh=dm)
        got = r.matrix()
        np.testing.assert_array_equal(got.col_ptr, a.col_ptr)
        assert _bits(got.values) == _bits(a.values)
        np.testing.assert_array_equal(r.partition().free_nodes, f)
        np.testing.assert_array_equal(r.partition().dirichlet_nodes, d)
        aff = po.submatrix(a, f, f, which=ref_which)
        assert _bits(r.matrix_ff().values) == _bits(aff.values)


@pytest.mark.parametrize("world", [1, 3])
def test_result_counts_async_matches_sizes(world, ctx):
    """fl_result_counts_async (the payload of the NCCL nnz-offset exchange)."""
    import ctypes as C
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cube3_mixed_jit.npz"))
    m = _mesh(g)
    for r in range(world):
        sa = ShardedAssembler(m, r, world, ctx=ctx)
        res = sa.assemble(_lib.OUT_SYSTEM, f=1.0, g_dirichlet=0.0)
        s = res.sizes()
        import torch
        out = torch.zeros(4, dtype=torch.int64, device="cuda")
        ctx.synchronize()
        _lib.check(_lib.lib().fl_result_counts_async(res.handle, C.c_void_p(out.data_ptr())))
        ctx.synchronize()
        assert out.cpu().tolist() == [s.n, s.n_free_cols, s.nnz, s.nnz_ff]


def test_bench_two_ranks_gather_gloo(tmp_path, ref_which):
    """bench.py --gpus 2 under torchrun on ONE GPU with FL_BENCH_BACKEND=gloo (a
    functional check of the sharded path: both ranks share cuda:0, so the numbers
    mean nothing): the grouped send/recv verification gather to rank 0
    (shard.gather_csc_to_root, NCCL on a real multi-GPU run) reassembles the
    reference's A bit for bit."""
    import os
    import socket
    import subprocess
    import sys
    from paper_1804_05156_b200 import configs
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "gathered.npz"
    env = dict(os.environ, FL_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--config", "C2", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
           "--no-cached", "--dump-gather", str(out)]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    g = np.load(out)
    m = configs.build("C2").mesh
    a = po.assemble_blockwise(m.dim, m.nodes, m.elems, which=ref_which)
    np.testing.assert_array_equal(g["col_ptr"], a.col_ptr)
    np.testing.assert_array_equal(g["row_idx"], a.row_idx)
    assert g["values"].tobytes() == a.values.tobytes()
