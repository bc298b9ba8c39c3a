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


@pytest.mark.parametrize("dim,npts,seed,cluster", [(2, 3000, 1, 0), (2, 2000, 2, 400), (3, 1500, 3, 0),
                                                   (3, 800, 4, 300)])
def test_unstructured_bitwise(dim, npts, seed, cluster, ctx, ref_which):
    m = _delaunay(dim, npts, seed, cluster)
    assert po.validate_mesh(m.dim, m.nodes, m.elems, m.bd_flags, which=ref_which) == 0
    ref = po.assemble_blockwise(m.dim, m.nodes, m.elems, which=ref_which)
    s = fl.poisson_system(m, 1.0, "x", ctx=ctx)
    np.testing.assert_array_equal(s.a.col_ptr, ref.col_ptr)
    np.testing.assert_array_equal(s.a.row_idx, ref.row_idx)
    assert s.a.values.tobytes() == ref.values.tobytes()
    b = po.assemble_load(m.dim, m.nodes, m.elems, po.FIELD_CONST, 1.0, which=ref_which)
    assert s.b.tobytes() == b.tobytes()
    u0, bm = po.apply_dirichlet(m.dim, m.nodes, m.elems, m.bd_flags, ref, b, po.FIELD_X, 0.0,
                                which=ref_which)
    assert s.b_mod.tobytes() == bm.tobytes()
    # the device-side classification of this mesh's boundary as well
    from paper_1804_05156_b200 import boundary
    g = boundary.set_boundary_flags(Mesh(m.dim, m.nodes, m.elems), fl.classifier_dirichlet, ctx=ctx)
    np.testing.assert_array_equal(g.bd_flags, m.bd_flags)
