"""Parity at BASELINE.json's full sizes (SURVEY.md §8 size sheet), through checks
that do not need the reference's full O(NT log) CPU assembly:

* exact counts: nnz, nnz_ff and the Dirichlet node count against the closed
  forms of the size sheet (square: (n+1)^2 + 4n(n+1); Kuhn cube:
  (n+1)^3 + 6n(n+1)^2; free blocks with n+1 -> n-1; C2 = its mesh graph);
* CSC invariants: col_ptr monotone, rows strictly increasing in every column;
* sampled columns bitwise against the C oracle's per-column restatement of
  assemble_blockwise (fo_assemble_columns: every element touching the column,
  the reference's (i(d+1)+j, t) fold order), the C5 coefficient given as host
  samples so the comparison is bitwise;
* the whole load vector and the Dirichlet / free node lists bitwise against
  the oracle (O(NT) passes), b_f = b_mod[free], A(free, free) columns = the
  sampled A columns filtered to free rows and renumbered;
* sum(b) = the domain measure for f = 1 (1e-12 relative).
Marked slow (each builds its mesh on the host first: up to ~20 s for C5).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from paper_1804_05156_b200 import _lib, configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

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


def _check_csc(a):
    cp, ri = a.col_ptr.astype(np.int64), a.row_idx
    assert cp[0] == 0 and np.all(np.diff(cp) >= 0) and cp[-1] == ri.size
    d = np.diff(ri.astype(np.int64))
    starts = cp[1:-1][(cp[1:-1] > 0) & (cp[1:-1] < ri.size)]  # first entry of a column
    ok = d > 0
    ok[starts - 1] = True  # a column boundary may go down
    assert ok.all(), "rows not strictly increasing inside a column"
    assert ri.min(initial=0) >= 0 and ri.max(initial=0) < a.m


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_config(name, ctx):
    f_mode = "samples" if name == "C2" else "kind"
    cfg = configs.build(name, f_mode=f_mode)
    m = cfg.mesh
    d, N, NT = m.dim, m.num_nodes(), m.num_elems()
    coef = configs.host_samples(m, rule=1, kind=_lib.FIELD_COEF_C5) if cfg.coef else None
    s = fl.poisson_system(m, cfg.f, 0.0, coef=coef, ctx=ctx)
    nnz, nnz_ff, n_dir = EXPECT[name]
    assert s.a.nnz() == nnz and s.a_ff.nnz() == nnz_ff
    assert s.partition.dirichlet_nodes.size == n_dir
    assert s.partition.free_nodes.size == N - n_dir
    _check_csc(s.a)
    _check_csc(s.a_ff)
    # node lists and the load vector: whole arrays, bitwise
    dn, fn = po.partition_boundary(d, m.nodes, m.elems, m.bd_flags)[:2]
    np.testing.assert_array_equal(s.partition.dirichlet_nodes, dn)
    np.testing.assert_array_equal(s.partition.free_nodes, fn)
    if isinstance(cfg.f, np.ndarray):
        b = po.assemble_load(d, m.nodes, m.elems, po.FIELD_SAMPLES, samples=cfg.f)
    else:
        b = po.assemble_load(d, m.nodes, m.elems, po.FIELD_CONST, float(cfg.f))
        measure = {"C1": 1.0, "C3": 1.0, "C4": 1.0, "C5": 1.0}[name]
        assert abs(float(np.sum(s.b)) - measure) <= 1e-12 * measure * 10
    assert (_bits(s.b) == _bits(b)).all()
    assert (_bits(s.b_f) == _bits(s.b_mod[fn])).all()
    # sampled columns of A, bitwise against the oracle; A(free,free) columns follow
    rng = np.random.default_rng(7)
    cols = np.unique(np.concatenate([rng.integers(0, N, 96), dn[:8], fn[:8], [0, N - 1]])).astype(np.int32)
    ref = po.assemble_columns(d, m.nodes, m.elems, cols, coef=coef)
    rank = np.full(N, -1, dtype=np.int64)
    rank[fn] = np.arange(fn.size)
    for k, c in enumerate(cols):
        g0, g1 = s.a.col_ptr[c], s.a.col_ptr[c + 1]
        r0, r1 = ref.col_ptr[k], ref.col_ptr[k + 1]
        np.testing.assert_array_equal(s.a.row_idx[g0:g1], ref.row_idx[r0:r1])
        assert (_bits(s.a.values[g0:g1]) == _bits(ref.values[r0:r1])).all(), (name, c)
        if rank[c] >= 0:
            rows, vals = s.a.row_idx[g0:g1], s.a.values[g0:g1]
            keep = rank[rows] >= 0
            f0, f1 = s.a_ff.col_ptr[rank[c]], s.a_ff.col_ptr[rank[c] + 1]
            np.testing.assert_array_equal(s.a_ff.row_idx[f0:f1], rank[rows[keep]])
            assert (_bits(s.a_ff.values[f0:f1]) == _bits(vals[keep])).all()
