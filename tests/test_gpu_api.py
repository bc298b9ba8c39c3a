"""GPU parity of the boundary entry points that take caller data:
apply_dirichlet(A, b, mesh, g) for an A and b that are NOT the assembled ones
(system.hpp:182-201), accumulate (sparse.hpp:186-198), and the FaceLists of
partition_boundary (mesh.hpp:222-246) -- all bitwise against the reference."""
import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from paper_1804_05156_b200 import _lib
from paper_1804_05156_b200.errors import Error, ErrorCode
from oracle import pyoracle as po

from .meshes import catalog

pytestmark = pytest.mark.gpu
MESHES = catalog()
DIRICHLET = sorted(k for k, m in MESHES.items() if np.any(m.bd_flags == 1))


def _random_matrix(n, rng, density=6):
    """A by from_triplets of random COO (duplicates, cancellations): not an assembled A."""
    cnt = density * n
    ii = rng.integers(0, n, cnt).astype(np.int32)
    jj = rng.integers(0, n, cnt).astype(np.int32)
    ss = rng.standard_normal(cnt) * 10.0 ** rng.integers(-3, 4, cnt)
    return po.from_triplets(n, n, ii, jj, ss, which="oracle")


@pytest.mark.parametrize("name", DIRICHLET)
@pytest.mark.parametrize("kind", ["twice_a", "triplets"])
@pytest.mark.parametrize("g", ["x", "const", "samples"])
def test_apply_dirichlet_caller_matrix(name, kind, g, ctx, ref_which):
    m = MESHES[name]
    n = m.num_nodes()
    rng = np.random.default_rng(n + len(kind))
    if kind == "twice_a":
        a = po.assemble_blockwise(m.dim, m.nodes, m.elems, which=ref_which)
        a = po.Csc(a.m, a.n, a.col_ptr, a.row_idx, 2.0 * a.values)
    else:
        a = _random_matrix(n, rng)
    b = rng.standard_normal(n)
    if g == "x":
        spec, gk, gv, gs = "x", po.FIELD_X, 0.0, None
    elif g == "const":
        spec, gk, gv, gs = 1.25, po.FIELD_CONST, 1.25, None
    else:
        gs = rng.standard_normal(n)
        spec, gk, gv = gs, po.FIELD_SAMPLES, 0.0
    if gk == po.FIELD_SAMPLES:
        # the reference takes callables: the C restatement evaluates the samples
        u0r, br = po.apply_dirichlet(m.dim, m.nodes, m.elems, m.bd_flags, a, b, gk, gv, gs, which="oracle")
    else:
        u0r, br = po.apply_dirichlet(m.dim, m.nodes, m.elems, m.bd_flags, a, b, gk, gv, which=ref_which)
    got = fl.apply_dirichlet(fl.CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values), b, m, spec, ctx=ctx)
    assert got.u0.tobytes() == u0r.tobytes(), name
    assert got.b.tobytes() == br.tobytes(), name
    d, f, ndf, nnf = po.partition_boundary(m.dim, m.nodes, m.elems, m.bd_flags, which=ref_which)
    assert np.array_equal(got.partition.dirichlet_nodes, d) and np.array_equal(got.partition.free_nodes, f)
    faces, parent, local = po.boundary_faces(m.dim, m.nodes, m.elems, m.bd_flags, 1, which=ref_which)
    assert np.array_equal(got.partition.dirichlet_faces.faces, faces)
    assert np.array_equal(got.partition.dirichlet_faces.parent_elem, parent)
    assert np.array_equal(got.partition.dirichlet_faces.local_face, local)


def test_apply_dirichlet_errors(ctx):
    m = MESHES[DIRICHLET[0]]
    n = m.num_nodes()
    a = po.assemble_blockwise(m.dim, m.nodes, m.elems, which="oracle")
    A = fl.CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values)
    with pytest.raises(Error) as e:  # b of the wrong length
        fl.apply_dirichlet(A, np.zeros(n + 1), m, 0.0, ctx=ctx)
    assert e.value.code() == ErrorCode.shape_mismatch
    # no Dirichlet faces: the reference checks that before the sizes
    m0 = fl.Mesh(m.dim, m.nodes, m.elems, np.zeros_like(m.bd_flags))
    with pytest.raises(Error) as e:
        fl.apply_dirichlet(A, np.zeros(n + 1), m0, 0.0, ctx=ctx)
    assert e.value.code() == ErrorCode.no_dirichlet_boundary
    # Robin flags are rejected by partition_boundary first
    fr = m.bd_flags.copy()
    fr[fr == 1] = 3
    fr.flat[np.flatnonzero(m.bd_flags == 1)[0]] = 1
    m3 = fl.Mesh(m.dim, m.nodes, m.elems, fr)
    with pytest.raises(Error) as e:
        fl.apply_dirichlet(A, np.zeros(n), m3, 0.0, ctx=ctx)
    assert e.value.code() == ErrorCode.unsupported_boundary_type


@pytest.mark.parametrize("n,size", [(0, 5), (1, 1), (5000, 37), (200000, 100000)])
def test_accumulate(n, size, ctx, ref_which):
    rng = np.random.default_rng(n)
    idx = rng.integers(0, size, n).astype(np.int32)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-9, 9, n)
    if n:
        vals[::5] = -0.0
        vals[1::11] = -vals[0::11][: vals[1::11].size]  # exact cancellations
    got = fl.accumulate(idx, vals, size, ctx=ctx)
    ref = po.accumulate(idx, vals, size, which=ref_which)
    assert got.tobytes() == ref.tobytes()


def test_accumulate_index_out_of_range(ctx):
    with pytest.raises(Error) as e:
        fl.accumulate(np.array([0, 4], np.int32), np.ones(2), 4, ctx=ctx)
    assert e.value.code() == ErrorCode.index_out_of_range
