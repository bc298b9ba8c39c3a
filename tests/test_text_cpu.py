"""CPU tests of the text-writer row: the C oracle's
write_matrix_market / write_mesh are pinned to the reference's own output
(tests/golden/text, written by tests/golden/make_text_golden.py from oracle/_ref),
and the golden "%.17g" cases agree with this host's glibc snprintf."""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np
import pytest

from oracle import pyoracle as po

HERE = os.path.dirname(os.path.abspath(__file__))
TEXT = os.path.join(HERE, "golden", "text")
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import jitter  # noqa: E402
from make_text_golden import MESHES  # noqa: E402


def golden_mesh(name):
    for nm, shape, n, cls, jit in MESHES:
        if nm == name:
            d, nodes, elems = po.generate_mesh(shape, n)
            flags = po.set_boundary_flags(d, nodes, elems, cls)
            if jit:
                nodes = jitter(d, nodes, elems, flags, seed=7)
            return d, nodes, elems, flags
    raise KeyError(name)


def read(name):
    with open(os.path.join(TEXT, name), "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", [m[0] for m in MESHES])
def test_oracle_writers_match_reference_golden(name):
    d, nodes, elems, flags = golden_mesh(name)
    a = po.assemble_blockwise(d, nodes, elems)
    assert po.write_matrix_market(a) == read(name + ".mtx")
    assert po.write_mesh(d, nodes, elems, flags) == read(name + ".mesh")


def test_oracle_reals_match_reference_golden():
    r = np.load(os.path.join(TEXT, "reals.npy"))
    col = po.Csc(r.size, 1, np.array([0, r.size], np.int32), np.arange(r.size, dtype=np.int32), r)
    assert po.write_matrix_market(col) == read("reals.mtx")


def test_golden_reals_are_glibc_snprintf():
    libc = ctypes.CDLL("libc.so.6")
    buf = ctypes.create_string_buffer(64)
    r = np.load(os.path.join(TEXT, "reals.npy"))
    lines = read("reals.mtx").decode().split("\n")[2:-1]
    assert len(lines) == r.size
    for v, line in zip(r, lines):
        libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
        assert line.split(" ")[2] == buf.value.decode()


def test_golden_reals_cover_ties_and_specials():
    r = np.load(os.path.join(TEXT, "reals.npy"))
    assert np.isnan(r).any() and np.isinf(r).any() and (r == 0).any()
    assert (np.abs(r[np.isfinite(r)]) < 2.3e-308).sum() >= 32  # subnormals
    # exact ties at the 17th digit: the exact decimal expansion has 18 digits ending in 5
    from decimal import Decimal
    ties = 0
    for v in r[np.isfinite(r) & (r != 0)]:
        t = Decimal(float(v)).normalize().as_tuple()
        if len(t.digits) == 18 and t.digits[-1] == 5:
            ties += 1
    assert ties >= 100
