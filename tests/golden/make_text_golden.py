"""Golden text fixtures written by the REFERENCE itself.

    python tests/golden/make_text_golden.py      (needs oracle/_ref, this container)

* text/<mesh>.mtx   write_matrix_market(assemble_blockwise(mesh))  matrix_market.hpp:15-24
* text/<mesh>.mesh  write_mesh(mesh)                               mesh_io.hpp:125-142
* text/reals.npy + text/reals.mtx: hard "%.17g" cases (exact decimal ties at
  the 17th digit, decade carries, subnormals, extremes, -0, inf, nan, random bit
  patterns) written by the reference's write_matrix_market as one CSC column.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import pyoracle as po  # noqa: E402
from make_golden import jitter  # noqa: E402

OUT = os.path.join(HERE, "text")
MESHES = [("square4_mixed_jit", po.SHAPE_SQUARE, 4, po.CLS_MIXED, True),
          ("lshape4", po.SHAPE_LSHAPE, 4, po.CLS_LSHAPE, False),
          ("cube3_mixed_jit", po.SHAPE_CUBE, 3, po.CLS_MIXED, True)]


def hard_reals(seed: int = 20261020) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = [0.0, -0.0, 1.0, -1.0, 0.1, 1 / 3, 2 / 3, 0.5, 1.5, 2.5, 1e-5, 1e-4, 9.9999999999999995e-5,
         1e16, 1e17, 12345678901234567.0, 123456789012345678.0, 2.0 ** 53, 2.0 ** 60, 5e-324,
         2.2250738585072014e-308, 2.2250738585072009e-308, 1.7976931348623157e308, 0.1 + 0.2,
         np.inf, -np.inf, np.nan, 100.0, 1e21, 1e22, 1e23, 123456.0, 1e-300, 4.35e-5, 9.5, 0.95]
    # exact ties at the 17th significant digit: odd * 2^-j with 18 significant digits
    for a in range(0, 17):  # v in [10^a, 10^(a+1)), j = 17 - a
        j = 17 - a
        lo, hi = int(np.ceil(10.0 ** a * 2 ** j)), int(10.0 ** (a + 1) * 2 ** j)
        for _ in range(6):
            m = int(rng.integers(lo, hi)) | 1
            v.append(m / 2.0 ** j)
            v.append((m + 2) / 2.0 ** j)
    for b in range(1, 9):  # v in [10^-b, 10^-b+1), j = 17 + b (empty range beyond b = 8)
        j = 17 + b
        lo, hi = max(int(np.ceil(10.0 ** -b * 2 ** j)), 1), int(10.0 ** (1 - b) * 2 ** j)
        if lo >= hi:
            continue
        for _ in range(4):
            m = int(rng.integers(lo, hi)) | 1
            v.append(m / 2.0 ** j)
    # around powers of ten (decade carries) over the whole range
    for k in range(-323, 309, 3):
        p = 10.0 ** k
        v += [p, np.nextafter(p, 0.0), np.nextafter(p, np.inf)]
    # subnormals, uniform bit patterns, integers, both signs
    v += list(rng.integers(1, 2 ** 52, size=64).astype(np.uint64).view(np.float64))
    bits = rng.integers(0, 0x7FF0000000000000, size=1500, dtype=np.int64).view(np.float64)
    v += list(bits)
    v += list(rng.integers(-10 ** 15, 10 ** 15, size=64).astype(np.float64))
    v += list(rng.standard_normal(200) * 10.0 ** rng.integers(-20, 20, size=200))
    out = np.array(v, dtype=np.float64)
    sign = rng.random(out.size) < 0.3
    out[sign] = -out[sign]
    return out


def main():
    assert po.have_ref(), "build oracle/_ref first (make -C oracle ref)"
    os.makedirs(OUT, exist_ok=True)
    for name, shape, n, cls, jit in MESHES:
        d, nodes, elems = po.generate_mesh(shape, n, which="ref")
        flags = po.set_boundary_flags(d, nodes, elems, cls, which="ref")
        if jit:
            nodes = jitter(d, nodes, elems, flags, seed=7)
        a = po.assemble_blockwise(d, nodes, elems, which="ref")
        with open(os.path.join(OUT, name + ".mtx"), "wb") as f:
            f.write(po.write_matrix_market(a, which="ref"))
        with open(os.path.join(OUT, name + ".mesh"), "wb") as f:
            f.write(po.write_mesh(d, nodes, elems, flags, which="ref"))
    r = hard_reals()
    np.save(os.path.join(OUT, "reals.npy"), r)
    col = po.Csc(r.size, 1, np.array([0, r.size], np.int32), np.arange(r.size, dtype=np.int32), r)
    with open(os.path.join(OUT, "reals.mtx"), "wb") as f:
        f.write(po.write_matrix_market(col, which="ref"))


if __name__ == "__main__":
    main()
