"""GPU: the solve after the path against the reference's
matvec / cg_solve / solve_poisson (oracle/_ref).

matvec is bitwise (row sums in the reference's column order).  CG's dot
products are deterministic tree reductions, not the reference's sequential
sums, so CG is compared by tolerance: both stop at |r| <= rel_tol |b|, the
solutions agree to SOLVE_TOL relative, and iteration counts agree within 2.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from paper_1804_05156_b200 import configs
from paper_1804_05156_b200.api import CscMatrix
from paper_1804_05156_b200.mesh import Mesh

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not po.have_ref(), reason="oracle/_ref not built")]
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SOLVE_TOL = 1e-7  # relative max-norm difference of two rel_tol = 1e-10 CG solutions


def _aff(tag):
    g = np.load(os.path.join(GOLD, tag + ".npz"))
    a = po.Csc(int(g["free_nodes"].size), int(g["free_nodes"].size), g["aff_col_ptr"], g["aff_row_idx"],
               g["aff_values"])
    return g, a


@pytest.mark.parametrize("tag", ["square8_jit", "lshape4_jit", "cube3_mixed_jit", "cube2_jit"])
def test_matvec_bitwise(tag, ctx):
    g = np.load(os.path.join(GOLD, tag + ".npz"))
    n = g["a_col_ptr"].size - 1
    a = po.Csc(n, n, g["a_col_ptr"], g["a_row_idx"], g["a_values"])
    x = np.random.default_rng(1).standard_normal(n)
    got = fl.matvec(CscMatrix(n, n, a.col_ptr, a.row_idx, a.values), x, ctx=ctx)
    assert got.tobytes() == po.ref_matvec(a, x).tobytes()


@pytest.mark.parametrize("tag", ["square8_jit", "lshape4_jit", "cube3_mixed_jit"])
@pytest.mark.parametrize("precond", ["none", "jacobi"])
def test_cg_matches_reference(tag, precond, ctx):
    g, a = _aff(tag)
    b = g["bmod_x"][g["free_nodes"]]
    pc = {"none": 0, "jacobi": 1}[precond]
    xr, itr, rr, cr = po.ref_cg_solve(a, b, 1e-10, 0, pc)
    res = fl.cg_solve(CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values), b, 1e-10, 0, precond, ctx=ctx)
    assert res.converged and cr
    assert abs(res.iterations - itr) <= 2
    assert res.relres <= 1e-10
    assert np.max(np.abs(res.x - xr)) <= SOLVE_TOL * np.max(np.abs(xr))
    again = fl.cg_solve(CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values), b, 1e-10, 0, precond, ctx=ctx)
    assert again.x.tobytes() == res.x.tobytes()  # deterministic


def test_cg_edge_cases(ctx):
    g, a = _aff("square8_jit")
    A = CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values)
    z = fl.cg_solve(A, np.zeros(a.n), ctx=ctx)
    assert z.iterations == 0 and not np.any(z.x)
    b = g["bmod_x"][g["free_nodes"]]
    capped = fl.cg_solve(A, b, 1e-14, 3, "none", ctx=ctx)
    xr, itr, rr, cr = po.ref_cg_solve(a, b, 1e-14, 3, 0)
    assert not capped.converged and not cr and capped.iterations == itr == 3
    assert abs(capped.relres - rr) <= 1e-9 * rr
    neg = CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, -a.values)
    with pytest.raises(fl.Error) as e:
        fl.cg_solve(neg, b, ctx=ctx)
    assert e.value.code() == fl.ErrorCode.not_positive_definite
    with pytest.raises(fl.Error) as e:
        fl.cg_solve(A, b, rel_tol=0.0, ctx=ctx)
    assert e.value.code() == fl.ErrorCode.invalid_parameter


@pytest.mark.parametrize("name,n", [("C1", 24), ("C2", 16), ("C4", 8), ("C5", 6)])
def test_solve_poisson_matches_reference(name, n, ctx):
    cfg = configs.build(name, n=n)
    m = cfg.mesh
    f_kind, f_val = (po.FIELD_SINSIN, 0.0) if cfg.f == "sinsin" else (po.FIELD_CONST, float(cfg.f))
    if cfg.coef is not None:
        pytest.skip("the reference solve_poisson has no coefficient")
    ur, itr, rr, _ = po.ref_solve_poisson(m.dim, m.nodes, m.elems, m.bd_flags, f_kind, f_val,
                                          po.FIELD_X, 0.0)
    sol = fl.solve_poisson(m, cfg.f, "x", ctx=ctx)
    assert abs(sol.iterations - itr) <= 2
    assert np.max(np.abs(sol.u - ur)) <= SOLVE_TOL * max(1.0, np.max(np.abs(ur)))
    d = sol.partition.dirichlet_nodes
    assert sol.u[d].tobytes() == ur[d].tobytes()  # Dirichlet values are exact


@pytest.mark.parametrize("shape,n", [(0, 12), (1, 5)])
def test_solve_poisson_pure_neumann(shape, n, ctx):
    from paper_1804_05156_b200 import mesh as M
    m = M.set_boundary_flags(M.generate_mesh(M.MeshShape(shape), n), M.classifier_neumann)
    # a source with nonzero mean: enforce_compatibility projects it
    ur, itr, rr, _ = po.ref_solve_poisson(m.dim, m.nodes, m.elems, m.bd_flags, po.FIELD_X, 0.0,
                                          po.FIELD_CONST, 0.0)
    sol = fl.solve_poisson(m, "x", None, ctx=ctx)
    assert abs(sol.iterations - itr) <= 2
    assert np.max(np.abs(sol.u - ur)) <= SOLVE_TOL * max(1.0, np.max(np.abs(ur)))
