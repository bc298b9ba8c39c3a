"""Benchmark of SURVEY.md §8(f) row 2: solve_poisson (solver.hpp:223-247) end to
end on the GPU (assembly + Jacobi-CG on A(free,free) + nodal scatter, device-
resident, rel_tol 1e-10) vs the reference's own solve_poisson on a bounded
sample (oracle/_ref, 1 thread).  One JSON line per config.

  python tools/bench_solve.py [--config C4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_1804_05156_b200 import configs  # noqa: E402

SAMPLE_N = {"C1": 128, "C2": 128, "C3": 256, "C4": 32}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
cfg = configs.build(args.config)
m = cfg.mesh
ctx = fl.Context.default()
sol = fl.solve_poisson(m, cfg.f, 0.0, ctx=ctx)  # warm-up
ts = []
for _ in range(args.steps):
    t0 = time.perf_counter()
    sol = fl.solve_poisson(m, cfg.f, 0.0, ctx=ctx)
    ts.append(time.perf_counter() - t0)
sec = float(np.median(ts))
line = {"metric": "solve_poisson elements/s (GPU: assembly + Jacobi-CG + scatter)", "config": cfg.description,
        "n_elems": m.num_elems(), "n_free": int(sol.partition.free_nodes.size), "iterations": sol.iterations,
        "final_relres": sol.final_relres, "ms_per_solve": sec * 1e3, "value": m.num_elems() / sec,
        "unit": "elements/s", "timing": "wall clock, host mesh in, u out (includes H2D/D2H)"}
if po.have_ref() and args.config in SAMPLE_N:
    s = configs.build(args.config, n=SAMPLE_N[args.config])
    sm = s.mesh
    f_kind, f_val = (po.FIELD_SINSIN, 0.0) if s.f == "sinsin" else (po.FIELD_CONST, float(s.f))
    u, it, rr, secs = po.ref_solve_poisson(sm.dim, sm.nodes, sm.elems, sm.bd_flags, f_kind, f_val,
                                           po.FIELD_CONST, 0.0)
    g = fl.solve_poisson(sm, s.f, 0.0, ctx=ctx)
    line["cpu_baseline"] = {"value": sm.num_elems() / secs, "unit": "elements/s", "cores": 1,
                            "kind": "reference", "iterations": it,
                            "sample": f"{s.description} (n={SAMPLE_N[args.config]}, NT={sm.num_elems()}), "
                                      "femlite solve_poisson, 1 thread"}
    t0 = time.perf_counter()
    g = fl.solve_poisson(sm, s.f, 0.0, ctx=ctx)
    line["gpu_on_sample"] = {"ms": (time.perf_counter() - t0) * 1e3, "iterations": g.iterations,
                             "max_abs_diff_vs_reference": float(np.max(np.abs(g.u - u)))}
print(json.dumps(line))
