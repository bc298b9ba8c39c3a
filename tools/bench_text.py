"""Benchmark of SURVEY.md §8(f) row 4: the text writers on the GPU vs the
reference's writers (oracle/_ref, 1 thread).

    python tools/bench_text.py [CONFIG]      (default C4)

GPU: write_matrix_market of the assembled A straight from the device result
(device time, median of 5, CUDA-synchronised wall clock around the call; and
e2e = + the D2H copy of the text into pinned host memory), write_mesh of the
mesh's device arrays.  CPU: the reference's write_matrix_market / write_mesh
into an ostringstream on a bounded sample (unit_cube:32 / unit_square:256),
reported as bytes/s; outputs compared byte for byte on the sample.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_1804_05156_b200 import _lib, configs  # noqa: E402

PEAK = 6547.8e9
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = configs.build(name)
ctx = fl.Context.default()
r = fl.AssemblyResult(ctx)
fl.run(cfg.mesh, _lib.OUT_STIFFNESS, coef=cfg.coef, ctx=ctx, result=r)
s = r.sizes()
t = fl.Text(ctx)
L = _lib.lib()


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def mm():
    _lib.check(L.fl_write_matrix_market(ctx.handle, s.n, s.n, r.device_ptr(_lib.A_COL_PTR)[0],
                                        r.device_ptr(_lib.A_ROW_IDX)[0], r.device_ptr(_lib.A_VALUES)[0],
                                        _lib.MEM_DEVICE, t.handle))
    return t.size()


sec = timed(mm)
nbytes = t.size()
host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)


def mm_e2e():
    mm()
    _lib.check(L.fl_text_copy(t.handle, C.c_void_p(host.data_ptr()), nbytes, _lib.MEM_HOST))


sec_e2e = timed(mm_e2e)
in_bytes = 4 * (s.n + 1) + 12 * s.nnz
lines = [{"metric": "write_matrix_market bytes/s (GPU, device CSC -> device text)", "config": name,
          "nnz": int(s.nnz), "text_bytes": nbytes, "ms": sec * 1e3, "value": nbytes / sec,
          "unit": "bytes/s", "lines_per_s": s.nnz / sec,
          "hbm_gbs": (nbytes + in_bytes) / sec / 1e9, "hbm_frac": (nbytes + in_bytes) / sec / PEAK,
          "e2e": {"ms": sec_e2e * 1e3, "value": nbytes / sec_e2e, "unit": "bytes/s",
                  "d2h_bytes": nbytes}}]


def wm():
    _lib.check(L.fl_write_mesh(ctx.handle, cfg.mesh.device(ctx).handle, t.handle))
    return t.size()


sec_m = timed(wm, 3)
mbytes = t.size()
m = cfg.mesh
min_bytes = mbytes + m.nodes.nbytes + m.elems.nbytes + m.bd_flags.nbytes
lines.append({"metric": "write_mesh bytes/s (GPU, device mesh -> device text)", "config": name,
              "text_bytes": mbytes, "ms": sec_m * 1e3, "value": mbytes / sec_m, "unit": "bytes/s",
              "hbm_gbs": min_bytes / sec_m / 1e9, "hbm_frac": min_bytes / sec_m / PEAK})
if po.have_ref():
    for dim, shape, n in ((3, po.SHAPE_CUBE, 32), (2, po.SHAPE_SQUARE, 256)):
        d, nodes, elems = po.generate_mesh(shape, n, which="ref")
        flags = po.set_boundary_flags(d, nodes, elems, po.CLS_DIRICHLET, which="ref")
        nodes = nodes * (1.0 + 1e-3 * np.random.default_rng(1).random(nodes.shape))
        a = po.assemble_blockwise(d, nodes, elems, which="ref")
        txt, rs = po.write_matrix_market(a, which="ref", timing=True)
        g = fl.write_matrix_market(fl.CscMatrix(a.m, a.n, a.col_ptr, a.row_idx, a.values), ctx=ctx)
        mtxt, ms_ = po.write_mesh(d, nodes, elems, flags, which="ref", timing=True)
        gm = fl.write_mesh(fl.Mesh(d, nodes, elems, flags), ctx=ctx)
        lines.append({"metric": "reference CPU writers bytes/s (1 thread)", "sample": f"{shape}:{n}",
                      "write_matrix_market": {"value": len(txt) / rs, "unit": "bytes/s",
                                              "bytes": len(txt), "s": rs},
                      "write_mesh": {"value": len(mtxt) / ms_, "unit": "bytes/s", "bytes": len(mtxt),
                                     "s": ms_},
                      "cores": 1, "kind": "reference",
                      "gpu_bytes_equal": bool(g == txt and gm == mtxt)})
for ln in lines:
    print(json.dumps(ln))
