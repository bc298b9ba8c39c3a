"""CPU tests: pin the C oracle (oracle/femlite_oracle.c) to the reference.

1. Golden fixtures (tests/golden/*.npz, written by tests/golden/make_golden.py
   from the compiled reference): the oracle must reproduce every array bitwise.
2. Known-answer tests from the reference's own suite
   (sparse_test.cpp:36-70, assembly_test.cpp:42-148).
3. When oracle/_ref is built (this container), oracle == reference on extra
   random meshes, including the assemble_triplets strategy identity on the
   binary-fraction mesh (assembly_test.cpp:140-145).
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _csc_eq(a, col_ptr, row_idx, values):
    np.testing.assert_array_equal(a.col_ptr, col_ptr)
    np.testing.assert_array_equal(a.row_idx, row_idx)
    assert a.values.tobytes() == np.asarray(values, dtype=np.float64).tobytes()


def _bits_eq(x, y):
    assert np.asarray(x, dtype=np.float64).tobytes() == np.asarray(y, dtype=np.float64).tobytes()


def test_golden_fixtures_present():
    assert len(GOLDEN) >= 12


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_matches_golden(path):
    g = np.load(path)
    d, nodes, elems, flags = int(g["dim"]), g["nodes"], g["elems"], g["flags"]
    a = po.assemble_blockwise(d, nodes, elems)
    _csc_eq(a, g["a_col_ptr"], g["a_row_idx"], g["a_values"])
    for kind in (po.FIELD_CONST, po.FIELD_X, po.FIELD_XYZ, po.FIELD_SINSIN):
        value = 1.0 if kind == po.FIELD_CONST else 0.0
        _bits_eq(po.assemble_load(d, nodes, elems, kind, value), g[f"b_{kind}"])
    dn, fn, ndf, nnf = po.partition_boundary(d, nodes, elems, flags)
    np.testing.assert_array_equal(dn, g["dir_nodes"])
    np.testing.assert_array_equal(fn, g["free_nodes"])
    assert (ndf, nnf) == (int(g["n_dir_faces"]), int(g["n_neu_faces"]))
    b = g[f"b_{po.FIELD_CONST}"]
    u0, bm = po.apply_dirichlet(d, nodes, elems, flags, a, b, po.FIELD_X)
    _bits_eq(u0, g["u0_x"])
    _bits_eq(bm, g["bmod_x"])
    _bits_eq(po.apply_neumann(d, nodes, elems, flags, b, po.FIELD_CONST, 1.5), g["b_neumann_const15"])
    aff = po.submatrix(a, fn, fn)
    _csc_eq(aff, g["aff_col_ptr"], g["aff_row_idx"], g["aff_values"])
    coef = po.coefficient_c5(d, nodes, elems)
    _bits_eq(coef, g["coef"])
    ac = po.assemble_blockwise(d, nodes, elems, coef=coef)
    _csc_eq(ac, g["ac_col_ptr"], g["ac_row_idx"], g["ac_values"])


@pytest.mark.parametrize("path", GOLDEN[:4], ids=[os.path.basename(p)[:-4] for p in GOLDEN[:4]])
def test_oracle_column_subset_matches_golden(path):
    """fo_assemble_columns (the shard / spot-check path) == the golden columns."""
    g = np.load(path)
    d, nodes, elems = int(g["dim"]), g["nodes"], g["elems"]
    n = nodes.shape[0]
    cols = np.arange(n // 3, n, 2, dtype=np.int32)
    sub = po.assemble_columns(d, nodes, elems, cols)
    cp, ri, va = g["a_col_ptr"], g["a_row_idx"], g["a_values"]
    for k, c in enumerate(cols):
        lo, hi = sub.col_ptr[k], sub.col_ptr[k + 1]
        np.testing.assert_array_equal(sub.row_idx[lo:hi], ri[cp[c]:cp[c + 1]])
        _bits_eq(sub.values[lo:hi], va[cp[c]:cp[c + 1]])


# ---- known-answer tests of the reference suite ------------------------------------
def test_from_triplets_worked_example():  # sparse_test.cpp:36-43
    a = po.from_triplets(4, 3, [0, 1, 3, 1], [0, 1, 1, 2], [1.0, 2.0, 9.0, 4.0])
    assert (a.m, a.n) == (4, 3)
    np.testing.assert_array_equal(a.col_ptr, [0, 1, 3, 4])
    np.testing.assert_array_equal(a.row_idx, [0, 1, 3, 1])
    np.testing.assert_array_equal(a.values, [1.0, 2.0, 9.0, 4.0])


def test_from_triplets_duplicates_cancellation_tiny():  # sparse_test.cpp:45-70
    a = po.from_triplets(1, 1, [0, 0], [0, 0], [1.0, 2.0])
    assert a.nnz == 1 and a.values[0] == 3.0
    a = po.from_triplets(1, 1, [0, 0], [0, 0], [1.0, -1.0])
    assert a.nnz == 0
    np.testing.assert_array_equal(a.col_ptr, [0, 0])
    a = po.from_triplets(2, 2, [0, 1], [0, 1], [1e-300, 5e-324])
    assert a.nnz == 2 and a.values[0] == 1e-300 and a.values[1] == 5e-324


def test_from_triplets_rejects_bad_index():  # sparse_test.cpp:72-75
    with pytest.raises(po.OracleError):
        po.from_triplets(2, 2, [2], [0], [1.0])


@pytest.mark.parametrize("dim,verts,expected", [
    (2, [1.0, 0.0, 0.0, 1.0, 0.0, 0.0], [0.5, 0.0, -0.5, 0.0, 0.5, -0.5, -0.5, -0.5, 1.0]),
    (2, [0.0, 0.0, 1.0, 0.0, 0.0, 1.0], [1.0, -0.5, -0.5, -0.5, 0.5, 0.0, -0.5, 0.0, 0.5]),
    (3, [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1],
     [0.5, -1 / 6, -1 / 6, -1 / 6, -1 / 6, 1 / 6, 0, 0, -1 / 6, 0, 1 / 6, 0, -1 / 6, 0, 0, 1 / 6]),
])
def test_local_stiffness_kat(dim, verts, expected):  # assembly_test.cpp:42-62
    s, _ = po.local_stiffness_normals(dim, np.asarray(verts, dtype=np.float64))
    np.testing.assert_allclose(s.ravel(), expected, atol=1e-15, rtol=0)
    if po.have_ref():
        r, _ = po.local_stiffness_normals(dim, np.asarray(verts, dtype=np.float64), which="ref")
        _bits_eq(s, r)


def test_degenerate_simplex_rejected():  # assembly_test.cpp:99-103
    with pytest.raises(po.OracleError):
        po.local_stiffness_normals(2, np.array([0.0, 0.0, 1.0, 1.0, 2.0, 2.0]))


def _dense(a):
    out = np.zeros((a.m, a.n))
    for c in range(a.n):
        for k in range(a.col_ptr[c], a.col_ptr[c + 1]):
            out[a.row_idx[k], c] = a.values[k]
    return out


def test_unit_square_one_cell_hand_values():  # assembly_test.cpp:113-123, 165-178
    d, nodes, elems = po.generate_mesh(po.SHAPE_SQUARE, 1)
    a = po.assemble_blockwise(d, nodes, elems)
    np.testing.assert_array_equal(_dense(a), [[1.0, -0.5, -0.5, 0.0], [-0.5, 1.0, 0.0, -0.5],
                                              [-0.5, 0.0, 1.0, -0.5], [0.0, -0.5, -0.5, 1.0]])
    assert a.nnz == 12


def test_center_node_diagonal_is_four():  # assembly_test.cpp:125-140
    d, nodes, elems = po.generate_mesh(po.SHAPE_SQUARE, 2)
    a = po.assemble_blockwise(d, nodes, elems)
    assert abs(_dense(a)[4, 4] - 4.0) <= 1e-14


def test_row_sums_vanish():  # gradients of barycentric coordinates sum to 0
    d, nodes, elems = po.generate_mesh(po.SHAPE_CUBE, 3)
    a = _dense(po.assemble_blockwise(d, nodes, elems))
    assert np.max(np.abs(a.sum(axis=1))) <= 1e-13


# ---- oracle == reference (only where oracle/_ref was built) ------------------------
needs_ref = pytest.mark.skipif(not po.have_ref(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("shape,n", [(po.SHAPE_SQUARE, 13), (po.SHAPE_LSHAPE, 7), (po.SHAPE_CUBE, 4)])
def test_oracle_equals_reference_generated(shape, n):
    d, nodes, elems = po.generate_mesh(shape, n, which="ref")
    d2, nodes2, elems2 = po.generate_mesh(shape, n, which="oracle")
    np.testing.assert_array_equal(elems, elems2)
    _bits_eq(nodes, nodes2)
    rng = np.random.default_rng(n)
    nodes = nodes + rng.uniform(-0.02 / n, 0.02 / n, size=nodes.shape)
    a = po.assemble_blockwise(d, nodes, elems, which="ref")
    _csc_eq(po.assemble_blockwise(d, nodes, elems), a.col_ptr, a.row_idx, a.values)
    for kind in (po.FIELD_CONST, po.FIELD_SINSIN, po.FIELD_XYZ):
        _bits_eq(po.assemble_load(d, nodes, elems, kind, 2.0),
                 po.assemble_load(d, nodes, elems, kind, 2.0, which="ref"))


@needs_ref
def test_reference_blockwise_equals_triplets_on_binary_mesh():  # assembly_test.cpp:140-145
    d, nodes, elems = po.generate_mesh(po.SHAPE_SQUARE, 8, which="ref")
    a = po.ref_assemble_strategy(d, nodes, elems, 2)
    b = po.ref_assemble_strategy(d, nodes, elems, 1)
    _csc_eq(a, b.col_ptr, b.row_idx, b.values)


@needs_ref
@pytest.mark.parametrize("path", GOLDEN)
def test_oracle_face_lists_equal_reference(path):
    """boundary_faces (mesh.hpp:222-246): the C restatement == the reference."""
    g = np.load(path)
    d, nodes, elems, flags = int(g["dim"]), g["nodes"], g["elems"], g["flags"]
    for value in (1, 2):
        a = po.boundary_faces(d, nodes, elems, flags, value)
        b = po.boundary_faces(d, nodes, elems, flags, value, which="ref")
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
        assert a[0].shape[1] == d


@needs_ref
def test_oracle_accumulate_equals_reference():
    """accumulate (sparse.hpp:186-198): order-sensitive sums and signed zeros."""
    rng = np.random.default_rng(7)
    idx = rng.integers(0, 50, size=4000).astype(np.int32)
    vals = rng.standard_normal(4000) * 10.0 ** rng.integers(-8, 9, size=4000)
    vals[::7] = -0.0
    a = po.accumulate(idx, vals, 60)
    b = po.accumulate(idx, vals, 60, which="ref")
    assert a.tobytes() == b.tobytes()
    with pytest.raises(po.OracleError):
        po.accumulate(np.array([3, 70], np.int32), np.ones(2), 60, which="ref")
