"""Benchmark of SURVEY.md §8(f) row 1: set_boundary_flags (mesh.hpp:251-304) on
the GPU vs the reference's own CPU implementation (oracle/_ref).

  python tools/bench_boundary.py [--config C3] [--steps 5]

GPU step: topology plan + boundary-face matching + centroids + count read-back
+ flag scatter with the configs' classifier (all faces Dirichlet), device-
resident mesh, wall clock around the synchronising calls.  The reference runs
on a bounded sample of the same config family (1 thread, as written).
One JSON line.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib, configs  # noqa: E402
from paper_1804_05156_b200.mesh import DeviceMesh, Mesh  # noqa: E402

SAMPLE_N = {"C1": 128, "C2": 256, "C3": 1024, "C4": 48, "C5": 48}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
cfg = configs.build(args.config)
m = Mesh(cfg.mesh.dim, cfg.mesh.nodes, cfg.mesh.elems)
ctx = fl.Context.default()
L = _lib.lib()
dm = DeviceMesh(ctx, m)
n = C.c_int64()


def step():
    _lib.check(L.fl_mesh_plan(ctx.handle, dm.handle))
    _lib.check(L.fl_boundary_faces(ctx.handle, dm.handle, C.byref(n)))
    _lib.check(L.fl_mesh_set_boundary_flags(ctx.handle, dm.handle, None, 1, _lib.MEM_HOST))
    ctx.synchronize()


for _ in range(2):
    step()
ts = []
for _ in range(args.steps):
    t0 = time.perf_counter()
    step()
    ts.append(time.perf_counter() - t0)
sec = float(np.median(ts))
line = {"metric": "set_boundary_flags faces/s (GPU, device-resident mesh)", "config": cfg.description,
        "n_elems": m.num_elems(), "faces": m.num_elems() * (m.dim + 1), "boundary_faces": int(n.value),
        "ms_per_step": sec * 1e3, "value": m.num_elems() * (m.dim + 1) / sec, "unit": "faces/s"}
from oracle import pyoracle as po  # noqa: E402
if po.have_ref():
    s = configs.build(args.config, n=SAMPLE_N[args.config])
    sm = s.mesh
    po.set_boundary_flags(sm.dim, sm.nodes, sm.elems, po.CLS_DIRICHLET, which="ref")
    rt = []
    for _ in range(3):
        t0 = time.perf_counter()
        po.set_boundary_flags(sm.dim, sm.nodes, sm.elems, po.CLS_DIRICHLET, which="ref")
        rt.append(time.perf_counter() - t0)
    r = float(np.median(rt))
    line["cpu_baseline"] = {"value": sm.num_elems() * (sm.dim + 1) / r, "unit": "faces/s", "cores": 1,
                            "kind": "reference", "sample": f"{s.description} (n={SAMPLE_N[args.config]}, "
                            f"NT={sm.num_elems()}), femlite set_boundary_flags, 1 thread"}
print(json.dumps(line))
