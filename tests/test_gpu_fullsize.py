"""Parity at BASELINE.json's full sizes (SURVEY.md §8 size sheet).

C1-C4: WHOLE arrays against the reference itself (oracle/_ref: femlite compiled
from its headers, 1 thread, <= ~40 s and ~11 GB per config on the host):

* A = assemble_blockwise(mesh): col_ptr, row_idx, values bitwise;
* b = assemble_load(mesh, f) bitwise (C2: f sampled on the host with glibc sin);
* u0, b - A u0 = apply_dirichlet(A, b, mesh, g) bitwise, for g = 0 and, on C1
  and C4, for g = x (the lift path at scale);
* A(free, free) = submatrix(A, free, free) and b_f bitwise;
* partition_boundary: Dirichlet / free node lists and both FaceLists.

C5 (100.7M elements; the reference would need ~50 GB and ~2 min): the exact
counts of the size sheet plus >= 10k columns bitwise against the reference run
on the sub-mesh of every element touching them (same node array, elements in
their original order, the coefficient as host samples), which assembles those
columns exactly as the whole mesh does; the whole load vector and node lists
against the C restatement.
Marked slow (each builds its mesh on the host first: up to ~20 s for C5).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from paper_1804_05156_b200 import _lib, configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
needs_ref = pytest.mark.skipif(not po.have_ref(), reason="oracle/_ref not built")

SQUARE = lambda n: (n + 1) ** 2 + 4 * n * (n + 1)  # noqa: E731
CUBE = lambda n: (n + 1) ** 3 + 6 * n * (n + 1) ** 2  # noqa: E731
EXPECT = {  # (nnz, nnz_ff, n_dir) -- SURVEY.md §8 size sheet
    "C1": (SQUARE(128), 80137, 512),
    "C2": (5511169, 5489674, 3073),
    "C3": (SQUARE(4096), 83828745, 16384),
    "C4": (14926977, 14241907, 98306),
    "C5": (118425857, 115679475, 393218),
}


def _bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def _csc_bitwise(got, ref, what):
    np.testing.assert_array_equal(got.col_ptr, ref.col_ptr, err_msg=f"{what}: col_ptr")
    np.testing.assert_array_equal(got.row_idx, ref.row_idx, err_msg=f"{what}: row_idx")
    same = _bits(got.values) == _bits(ref.values)
    assert same.all(), f"{what}: {(~same).sum()} values differ"


def _check_csc(a):
    cp, ri = a.col_ptr.astype(np.int64), a.row_idx
    assert cp[0] == 0 and np.all(np.diff(cp) >= 0) and cp[-1] == ri.size
    d = np.diff(ri.astype(np.int64))
    starts = cp[1:-1][(cp[1:-1] > 0) & (cp[1:-1] < ri.size)]  # first entry of a column
    ok = d > 0
    ok[starts - 1] = True  # a column boundary may go down
    assert ok.all(), "rows not strictly increasing inside a column"
    assert ri.min(initial=0) >= 0 and ri.max(initial=0) < a.m


@needs_ref
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_full_config_whole_arrays(name, ctx):
    f_mode = "samples" if name == "C2" else "kind"
    cfg = configs.build(name, f_mode=f_mode)
    m = cfg.mesh
    d, N = m.dim, m.num_nodes()
    g_cases = [(0.0, po.FIELD_CONST, 0.0)] + ([("x", po.FIELD_X, 0.0)] if name in ("C1", "C4") else [])
    # the reference, once per config
    A = po.assemble_blockwise(d, m.nodes, m.elems, which="ref")
    if isinstance(cfg.f, np.ndarray):
        # C2: the reference's own f = sin(pi x) sin(pi y) at its midpoints equals the
        # host samples bit for bit (tests/test_gpu_parity.py::test_load_sinsin)
        b = po.assemble_load(d, m.nodes, m.elems, po.FIELD_SINSIN, which="ref")
    else:
        b = po.assemble_load(d, m.nodes, m.elems, po.FIELD_CONST, float(cfg.f), which="ref")
    dn, fn, ndf, nnf = po.partition_boundary(d, m.nodes, m.elems, m.bd_flags, which="ref")
    Aff = po.submatrix(A, fn, fn, which="ref")
    nnz, nnz_ff, n_dir = EXPECT[name]
    assert A.nnz == nnz and Aff.nnz == nnz_ff and dn.size == n_dir
    faces = {v: po.boundary_faces(d, m.nodes, m.elems, m.bd_flags, v, which="ref") for v in (1, 2)}
    for gspec, gk, gv in g_cases:
        s = fl.poisson_system(m, cfg.f, gspec, ctx=ctx)
        u0, bmod = po.apply_dirichlet(d, m.nodes, m.elems, m.bd_flags, A, b, gk, gv, which="ref")
        what = f"{name} g={gspec}"
        _csc_bitwise(s.a, A, what + " A")
        _csc_bitwise(s.a_ff, Aff, what + " A(free,free)")
        assert (_bits(s.b) == _bits(b)).all(), what + " b"
        assert (_bits(s.u0) == _bits(u0)).all(), what + " u0"
        assert (_bits(s.b_mod) == _bits(bmod)).all(), what + " b - A u0"
        assert (_bits(s.b_f) == _bits(bmod[fn])).all(), what + " b_f"
        np.testing.assert_array_equal(s.partition.dirichlet_nodes, dn)
        np.testing.assert_array_equal(s.partition.free_nodes, fn)
        for v, fl_got in ((1, s.partition.dirichlet_faces), (2, s.partition.neumann_faces)):
            np.testing.assert_array_equal(fl_got.faces, faces[v][0])
            np.testing.assert_array_equal(fl_got.parent_elem, faces[v][1])
            np.testing.assert_array_equal(fl_got.local_face, faces[v][2])


@pytest.mark.parametrize("name", ["C5"])
def test_full_config_sampled(name, ctx):
    cfg = configs.build(name)
    m = cfg.mesh
    d, N = m.dim, m.num_nodes()
    coef = configs.host_samples(m, rule=1, kind=_lib.FIELD_COEF_C5)
    assert coef.tobytes() == po.coefficient_c5(d, m.nodes, m.elems).tobytes()
    s = fl.poisson_system(m, cfg.f, 0.0, coef=coef, ctx=ctx)
    nnz, nnz_ff, n_dir = EXPECT[name]
    assert s.a.nnz() == nnz and s.a_ff.nnz() == nnz_ff
    assert s.partition.dirichlet_nodes.size == n_dir
    _check_csc(s.a)
    _check_csc(s.a_ff)
    # node lists and the load vector: whole arrays, bitwise (the C restatement,
    # pinned against the reference in test_oracle_golden.py)
    dn, fn = po.partition_boundary(d, m.nodes, m.elems, m.bd_flags)[:2]
    np.testing.assert_array_equal(s.partition.dirichlet_nodes, dn)
    np.testing.assert_array_equal(s.partition.free_nodes, fn)
    b = po.assemble_load(d, m.nodes, m.elems, po.FIELD_CONST, float(cfg.f))
    assert (_bits(s.b) == _bits(b)).all()
    assert abs(float(np.sum(s.b)) - 1.0) <= 1e-11
    assert (_bits(s.b_f) == _bits(s.b_mod[fn])).all()
    # >= 10k columns against the reference on the sub-mesh of their elements
    rng = np.random.default_rng(7)
    cols = np.unique(np.concatenate([rng.integers(0, N, 10240), dn[:64], fn[:64], [0, N - 1]])).astype(np.int32)
    assert cols.size >= 10000
    touch = np.zeros(N, dtype=bool)
    touch[cols] = True
    sel = np.nonzero(touch[m.elems].any(axis=1))[0]  # ascending: the original element order
    A = po.assemble_blockwise(d, m.nodes, m.elems[sel], coef=coef[sel], which="ref" if po.have_ref() else "oracle")
    rank = np.full(N, -1, dtype=np.int64)
    rank[fn] = np.arange(fn.size)
    for c in cols:
        g0, g1 = s.a.col_ptr[c], s.a.col_ptr[c + 1]
        r0, r1 = A.col_ptr[c], A.col_ptr[c + 1]
        np.testing.assert_array_equal(s.a.row_idx[g0:g1], A.row_idx[r0:r1])
        assert (_bits(s.a.values[g0:g1]) == _bits(A.values[r0:r1])).all(), (name, c)
        if rank[c] >= 0:
            rows, vals = s.a.row_idx[g0:g1], s.a.values[g0:g1]
            keep = rank[rows] >= 0
            f0, f1 = s.a_ff.col_ptr[rank[c]], s.a_ff.col_ptr[rank[c] + 1]
            np.testing.assert_array_equal(s.a_ff.row_idx[f0:f1], rank[rows[keep]])
            assert (_bits(s.a_ff.values[f0:f1]) == _bits(vals[keep])).all()
