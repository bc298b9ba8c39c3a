"""GPU parity of the text writers: byte-identical to
the reference's write_matrix_market / write_mesh (golden fixtures written by
oracle/_ref) and to glibc's "%.17g" on hard and random doubles, through the
fast rounding path and the forced exact big-integer path."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po
from tests.test_text_cpu import MESHES, TEXT, golden_mesh, read

pytestmark = pytest.mark.gpu

_libc = ctypes.CDLL("libc.so.6")


def glibc_g17(values):
    buf = ctypes.create_string_buffer(64)
    out = []
    for v in values:
        _libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(float(v)))
        out.append(buf.value.decode())
    return out


@pytest.mark.parametrize("exact", [False, True])
def test_format_reals_golden(ctx, exact):
    r = np.load(os.path.join(TEXT, "reals.npy"))
    want = [ln.split(" ")[2] for ln in read("reals.mtx").decode().split("\n")[2:-1]]
    assert fl.format_reals(r, exact=exact, ctx=ctx) == want


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("exact", [False, True])
def test_format_reals_random_bits(ctx, seed, exact):
    rng = np.random.default_rng(seed)
    n = 60000 if not exact else 20000
    v = rng.integers(0, 2 ** 64 - 1, size=n, dtype=np.uint64).view(np.float64)  # incl. nan/inf
    v = np.concatenate([v, rng.standard_normal(n // 4), rng.integers(-10 ** 6, 10 ** 6, n // 4) / 8.0])
    assert fl.format_reals(v, exact=exact, ctx=ctx) == glibc_g17(v)


def test_format_reals_empty(ctx):
    assert fl.format_reals(np.zeros(0), ctx=ctx) == []


@pytest.mark.parametrize("name", [m[0] for m in MESHES])
def test_writers_match_reference_golden(ctx, name):
    d, nodes, elems, flags = golden_mesh(name)
    m = fl.Mesh(d, nodes, elems, flags)
    a = fl.assemble_blockwise(m, ctx=ctx)
    assert fl.write_matrix_market(a, ctx=ctx) == read(name + ".mtx")
    assert fl.write_mesh(m, ctx=ctx) == read(name + ".mesh")
    # straight from the device result of the assembly
    r = fl.AssemblyResult(ctx)
    fl.run(m, 1, ctx=ctx, result=r)
    assert fl.write_result_matrix_market(r) == read(name + ".mtx")


def test_writers_match_reference_larger_meshes(ctx, ref_which):
    for shape, n in ((po.SHAPE_SQUARE, 48), (po.SHAPE_CUBE, 9), (po.SHAPE_LSHAPE, 16)):
        d, nodes, elems = po.generate_mesh(shape, n)
        flags = po.set_boundary_flags(d, nodes, elems, po.CLS_MIXED if shape != po.SHAPE_LSHAPE
                                      else po.CLS_LSHAPE)
        rng = np.random.default_rng(n)
        nodes = nodes * (1.0 + 1e-3 * rng.random(nodes.shape))  # generic digits
        a = po.assemble_blockwise(d, nodes, elems, which="oracle")
        m = fl.Mesh(d, nodes, elems, flags)
        assert fl.write_matrix_market(fl.CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values),
                                      ctx=ctx) == po.write_matrix_market(a, which=ref_which)
        assert fl.write_mesh(m, ctx=ctx) == po.write_mesh(d, nodes, elems, flags, which=ref_which)


def test_matrix_market_ragged_and_empty(ctx, ref_which):
    # empty columns (ragged CSC), a 0 x 0 matrix, a matrix with no entries
    rng = np.random.default_rng(5)
    m, n = 50, 700
    cnt = rng.integers(0, 3, size=n) * (rng.random(n) < 0.3)
    cp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    ri = np.concatenate([np.sort(rng.choice(m, size=c, replace=False)) for c in cnt]).astype(np.int32)
    va = rng.standard_normal(ri.size) * 10.0 ** rng.integers(-30, 30, ri.size)
    for (mm, nn, c, r, v) in ((m, n, cp, ri, va), (0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32),
                                                   np.zeros(0)),
                              (3, 4, np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0))):
        want = po.write_matrix_market(po.Csc(mm, nn, c, r, v), which=ref_which)
        assert fl.write_matrix_market(fl.CscMatrix(mm, nn, c, r, v), ctx=ctx) == want
