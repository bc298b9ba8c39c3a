"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Run in the container that has /root/reference (oracle/_ref/libfemlite_ref.so is
the unmodified femlite headers compiled by oracle/Makefile):

    python tests/golden/make_golden.py

Each fixture is the reference's own output on a small mesh: assemble_blockwise
(CSC), assemble_load for several sources, partition_boundary, apply_dirichlet,
apply_neumann and submatrix(A, free, free), plus the known-answer cases its
test suite pins (sparse_test.cpp:36-70, assembly_test.cpp:42-62,
system_test.cpp:29-87).  The CPU tests check the C oracle against these files
and the GPU tests check the B200 path against them, so parity never depends on
/root/reference at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402

MESHES = [  # (name, shape, n, classifier)
    ("square1", po.SHAPE_SQUARE, 1, po.CLS_DIRICHLET),
    ("square4_mixed", po.SHAPE_SQUARE, 4, po.CLS_MIXED),
    ("square8", po.SHAPE_SQUARE, 8, po.CLS_DIRICHLET),
    ("lshape4", po.SHAPE_LSHAPE, 4, po.CLS_LSHAPE),
    ("cube2", po.SHAPE_CUBE, 2, po.CLS_DIRICHLET),
    ("cube3_mixed", po.SHAPE_CUBE, 3, po.CLS_MIXED),
]


def jitter(dim, nodes, elems, flags, seed):
    """Interior-node jitter (as configs C2) to get generic, non-binary values."""
    rng = np.random.default_rng(seed)
    nv = dim + 1
    on = np.zeros(nodes.shape[0], dtype=bool)
    t, lf = np.nonzero(flags > 0)
    for k in range(nv):
        sel = lf != k
        on[elems[t[sel], k]] = True
    h = np.max(np.abs(nodes[elems[:, 1]] - nodes[elems[:, 0]]))
    out = nodes.copy()
    out[~on] += rng.uniform(-0.15 * h, 0.15 * h, size=(int((~on).sum()), dim))
    return out


def main():
    assert po.have_ref(), "build oracle/_ref first (make -C oracle ref)"
    for name, shape, n, cls in MESHES:
        for jit in (False, True):
            d, nodes, elems = po.generate_mesh(shape, n, which="ref")
            flags = po.set_boundary_flags(d, nodes, elems, cls, which="ref")
            tag = name
            if jit:
                nodes = jitter(d, nodes, elems, flags, seed=n)
                assert po.validate_mesh(d, nodes, elems, flags, which="ref") == 0
                tag = name + "_jit"
            a = po.assemble_blockwise(d, nodes, elems, which="ref")
            loads = {}
            for kind, value in [(po.FIELD_CONST, 1.0), (po.FIELD_X, 0.0), (po.FIELD_XYZ, 0.0),
                                (po.FIELD_SINSIN, 0.0)]:
                loads[f"b_{kind}"] = po.assemble_load(d, nodes, elems, kind, value, which="ref")
            dn, fn, ndf, nnf = po.partition_boundary(d, nodes, elems, flags, which="ref")
            b = loads[f"b_{po.FIELD_CONST}"]
            u0, bm = po.apply_dirichlet(d, nodes, elems, flags, a, b, po.FIELD_X, which="ref")
            bn = po.apply_neumann(d, nodes, elems, flags, b, po.FIELD_CONST, 1.5, which="ref")
            aff = po.submatrix(a, fn, fn, which="ref")
            coef = po.coefficient_c5(d, nodes, elems)
            ac = po.assemble_blockwise(d, nodes, elems, coef=coef, which="ref")
            np.savez_compressed(
                os.path.join(HERE, f"{tag}.npz"), dim=d, nodes=nodes, elems=elems, flags=flags,
                a_col_ptr=a.col_ptr, a_row_idx=a.row_idx, a_values=a.values,
                dir_nodes=dn, free_nodes=fn, n_dir_faces=ndf, n_neu_faces=nnf,
                u0_x=u0, bmod_x=bm, b_neumann_const15=bn,
                aff_col_ptr=aff.col_ptr, aff_row_idx=aff.row_idx, aff_values=aff.values,
                coef=coef, ac_col_ptr=ac.col_ptr, ac_row_idx=ac.row_idx, ac_values=ac.values,
                **loads)
            print(tag, "nnz", a.nnz, "nnz_ff", aff.nnz)


if __name__ == "__main__":
    main()
