"""GPU: set_boundary_flags' face matching on the device
against the reference (mesh.hpp:251-304): oracle/_ref's set_boundary_flags (or
the C oracle), the golden fixtures, and edge cases."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from paper_1804_05156_b200 import boundary, configs
from paper_1804_05156_b200 import mesh as M

from .meshes import fix_orientation

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
# the shim's classifier ids (oracle/ref_shim.cpp make_classifier) and their vectorised twins
CLS = {po.CLS_DIRICHLET: M.classifier_dirichlet, po.CLS_NEUMANN: M.classifier_neumann,
       po.CLS_MIXED: M.classifier_mixed, po.CLS_LSHAPE: M.classifier_lshape}


@pytest.mark.parametrize("tag,cls", [("square1", po.CLS_DIRICHLET), ("square4_mixed", po.CLS_MIXED),
                                     ("square8_jit", po.CLS_DIRICHLET), ("lshape4", po.CLS_LSHAPE),
                                     ("lshape4_jit", po.CLS_LSHAPE), ("cube2", po.CLS_DIRICHLET),
                                     ("cube3_mixed_jit", po.CLS_MIXED)])
def test_boundary_flags_match_golden(tag, cls, ctx):
    g = np.load(os.path.join(GOLD, tag + ".npz"))
    m = M.Mesh(int(g["dim"]), g["nodes"], g["elems"])
    out = boundary.set_boundary_flags(m, CLS[cls], ctx=ctx)
    np.testing.assert_array_equal(out.bd_flags.ravel(), g["flags"].ravel())


def _relabeled(m, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(m.num_nodes()).astype(np.int32)
    inv = np.argsort(perm)
    nodes = m.nodes[inv]
    elems = perm[m.elems]
    elems = elems[rng.permutation(m.num_elems())]
    return M.Mesh(m.dim, nodes, fix_orientation(m.dim, nodes, elems))


@pytest.mark.parametrize("shape,n,cls", [(0, 13, po.CLS_MIXED), (2, 9, po.CLS_LSHAPE),
                                         (1, 5, po.CLS_MIXED), (1, 4, po.CLS_DIRICHLET)])
@pytest.mark.parametrize("relabel", [False, True])
def test_boundary_flags_match_reference(shape, n, cls, relabel, ctx, ref_which):
    m = M.generate_mesh(M.MeshShape(shape), n)
    if relabel:
        m = _relabeled(m, n)
    want = po.set_boundary_flags(m.dim, m.nodes, m.elems, cls, which=ref_which)
    got = boundary.set_boundary_flags(m, CLS[cls], ctx=ctx)
    np.testing.assert_array_equal(got.bd_flags.ravel(), np.asarray(want).ravel())
    # centroids: the reference's arithmetic (vertex sum in face order from 0.0, / d)
    faces, cen = boundary.boundary_faces(m, ctx=ctx)
    table = M.TRI_FACES if m.dim == 2 else M.TET_FACES
    verts = m.elems[faces[:, 0][:, None], table[faces[:, 1]]]
    for c in range(m.dim):
        acc = np.zeros(faces.shape[0])
        for k in range(m.dim):
            acc = acc + m.nodes[verts[:, k], c]
        assert (acc / m.dim).tobytes() == cen[:, c].tobytes()
    # ascending (t, lf) order, each boundary face once
    key = faces[:, 0].astype(np.int64) * (m.dim + 1) + faces[:, 1]
    assert np.all(np.diff(key) > 0)


def test_constant_classifier_and_assembly_on_device_flags(ctx):
    cfg = configs.build("C4", n=6)
    m = M.Mesh(cfg.mesh.dim, cfg.mesh.nodes, cfg.mesh.elems)
    out = boundary.set_boundary_flags(m, 1, ctx=ctx)
    np.testing.assert_array_equal(out.bd_flags, cfg.mesh.bd_flags)
    # the cached device mesh carries the GPU-written flags into the assembly
    s_dev = fl.poisson_system(out, 1.0, 0.0, ctx=ctx)
    s_host = fl.poisson_system(cfg.mesh, 1.0, 0.0, ctx=ctx)
    assert s_dev.a_ff.values.tobytes() == s_host.a_ff.values.tobytes()
    np.testing.assert_array_equal(s_dev.partition.dirichlet_nodes, s_host.partition.dirichlet_nodes)


def test_single_element_and_empty(ctx):
    tri = M.Mesh(2, np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]))
    faces, cen = boundary.boundary_faces(tri, ctx=ctx)
    assert faces.tolist() == [[0, 0], [0, 1], [0, 2]]
    tet = M.Mesh(3, np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]), np.array([[0, 1, 2, 3]]))
    assert boundary.boundary_faces(tet, ctx=ctx)[0].shape == (4, 2)
    empty = M.Mesh(2, np.zeros((3, 2)), np.zeros((0, 3), dtype=np.int32))
    assert boundary.boundary_faces(empty, ctx=ctx)[0].shape == (0, 2)


def test_bad_classifier_value(ctx):
    m = M.generate_mesh(M.MeshShape.unit_square, 3)
    with pytest.raises(fl.Error) as e:
        boundary.set_boundary_flags(m, lambda x, y, z: np.full(x.shape, 5), ctx=ctx)
    assert e.value.code() == fl.ErrorCode.invalid_flag_value
