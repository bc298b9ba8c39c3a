"""GPU parity on unstructured meshes: random Delaunay triangulations and
tetrahedralisations (scipy.spatial) with irregular valences, including nodes
above the fast kernels' limits (the general-kernel fallback), against the
reference (oracle/_ref, else the C oracle).  Bitwise."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from paper_1804_05156_b200.mesh import Mesh

from .meshes import fix_orientation

pytestmark = pytest.mark.gpu
spatial = pytest.importorskip("scipy.spatial")


def _delaunay(dim, npts, seed, center_cluster=0):
    rng = np.random.default_rng(seed)
    pts = rng.random((npts, dim))
    if center_cluster:  # a dense ball of points: high-valence nodes
        c = 0.5 + 0.02 * rng.standard_normal((center_cluster, dim))
        pts = np.vstack([pts, c])
    tri = spatial.Delaunay(pts)
    elems = tri.simplices.astype(np.int32)
    # drop slivers (|measure| tiny) so the reference's degeneracy test passes
    X = pts[elems]
    if dim == 2:
        meas = 0.5 * np.abs((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 2, 1] - X[:, 0, 1]) -
                            (X[:, 2, 0] - X[:, 0, 0]) * (X[:, 1, 1] - X[:, 0, 1]))
    else:
        meas = np.abs(np.einsum("ij,ij->i", np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]),
                                X[:, 3] - X[:, 0])) / 6.0
    elems = elems[meas > 1e-9]
    used = np.unique(elems)
    remap = -np.ones(pts.shape[0], dtype=np.int64)
    remap[used] = np.arange(used.size)
    pts = pts[used]
    elems = remap[elems].astype(np.int32)
    elems = fix_orientation(dim, pts, elems)
    m = Mesh(dim, pts, elems)
    return fl.set_boundary_flags(m, fl.classifier_dirichlet)


@pytest.mark.parametrize("g", ["x", 0.0])  # lift (tiled kernel) / no lift (register + hybrid)
@pytest.mark.parametrize("dim,npts,seed,cluster", [(2, 3000, 1, 0), (2, 2000, 2, 400), (3, 1500, 3, 0),
                                                   (3, 800, 4, 300)])
def test_unstructured_bitwise(dim, npts, seed, cluster, g, ctx, ref_which):
    m = _delaunay(dim, npts, seed, cluster)
    assert po.validate_mesh(m.dim, m.nodes, m.elems, m.bd_flags, which=ref_which) == 0
    ref = po.assemble_blockwise(m.dim, m.nodes, m.elems, which=ref_which)
    s = fl.poisson_system(m, 1.0, g, ctx=ctx)
    np.testing.assert_array_equal(s.a.col_ptr, ref.col_ptr)
    np.testing.assert_array_equal(s.a.row_idx, ref.row_idx)
    assert s.a.values.tobytes() == ref.values.tobytes()
    b = po.assemble_load(m.dim, m.nodes, m.elems, po.FIELD_CONST, 1.0, which=ref_which)
    assert s.b.tobytes() == b.tobytes()
    gk, gv = (po.FIELD_X, 0.0) if g == "x" else (po.FIELD_CONST, 0.0)
    u0, bm = po.apply_dirichlet(m.dim, m.nodes, m.elems, m.bd_flags, ref, b, gk, gv, which=ref_which)
    assert s.b_mod.tobytes() == bm.tobytes()
    d, f, _, _ = po.partition_boundary(m.dim, m.nodes, m.elems, m.bd_flags, which=ref_which)
    aff = po.submatrix(ref, f, f, which=ref_which)
    np.testing.assert_array_equal(s.a_ff.col_ptr, aff.col_ptr)
    np.testing.assert_array_equal(s.a_ff.row_idx, aff.row_idx)
    assert s.a_ff.values.tobytes() == aff.values.tobytes()
    assert s.b_f.tobytes() == bm[f].tobytes()
    # the device-side classification of this mesh's boundary as well
    from paper_1804_05156_b200 import boundary
    g = boundary.set_boundary_flags(Mesh(m.dim, m.nodes, m.elems), fl.classifier_dirichlet, ctx=ctx)
    np.testing.assert_array_equal(g.bd_flags, m.bd_flags)


@pytest.mark.parametrize("world", [2, 3])
def test_unstructured_sharded_hybrid(world, ctx):
    """Column ranges over a mesh whose high-valence columns take the hybrid pass."""
    from paper_1804_05156_b200 import _lib
    from paper_1804_05156_b200.shard import ShardedAssembler, stitch_csc
    m = _delaunay(3, 800, 4, 300)
    ref = fl.poisson_system(m, 1.0, 0.0, ctx=ctx)
    parts = []
    for r in range(world):
        sa = ShardedAssembler(m, r, world, ctx=ctx)
        parts.append(sa.assemble(_lib.OUT_SYSTEM, f=1.0, g_dirichlet=0.0))
    a = stitch_csc(m.num_nodes(), [(p.matrix().col_ptr, p.matrix().row_idx, p.matrix().values) for p in parts])
    np.testing.assert_array_equal(a.col_ptr, ref.a.col_ptr)
    assert a.values.tobytes() == ref.a.values.tobytes()
    aff = stitch_csc(ref.a_ff.m, [(p.matrix_ff().col_ptr, p.matrix_ff().row_idx, p.matrix_ff().values)
                                  for p in parts])
    np.testing.assert_array_equal(aff.col_ptr, ref.a_ff.col_ptr)
    assert aff.values.tobytes() == ref.a_ff.values.tobytes()
    assert np.concatenate([p.vector(_lib.B_F) for p in parts]).tobytes() == ref.b_f.tobytes()


@pytest.mark.parametrize("dim,npts,seed,cluster", [(2, 2000, 7, 400), (3, 800, 8, 300)])
def test_unstructured_neumann_and_lift(dim, npts, seed, cluster, ctx, ref_which):
    """Neumann shares + Dirichlet lift on a mesh with hybrid-pass columns."""
    m = _delaunay(dim, npts, seed, cluster)
    m = fl.set_boundary_flags(Mesh(m.dim, m.nodes, m.elems), fl.classifier_mixed)
    ref = po.assemble_blockwise(m.dim, m.nodes, m.elems, which=ref_which)
    b = po.assemble_load(m.dim, m.nodes, m.elems, po.FIELD_CONST, 1.0, which=ref_which)
    bn = po.apply_neumann(m.dim, m.nodes, m.elems, m.bd_flags, b, po.FIELD_X, 0.0, which=ref_which)
    u0, bm = po.apply_dirichlet(m.dim, m.nodes, m.elems, m.bd_flags, ref, bn, po.FIELD_X, 0.0,
                                which=ref_which)
    s = fl.poisson_system(m, 1.0, "x", g_neumann="x", ctx=ctx)
    assert s.b.tobytes() == bn.tobytes()
    assert s.b_mod.tobytes() == bm.tobytes()
    assert s.a.values.tobytes() == ref.values.tobytes()
