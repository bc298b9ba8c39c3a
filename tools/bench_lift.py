"""assemble_system with nonzero Dirichlet data (the lift path) vs g = 0."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import configs  # noqa: E402

out = {}
for name in sys.argv[1:] or ["C4"]:
    cfg = configs.build(name)
    ctx = fl.Context.default()
    for g in (0.0, "x"):
        r = fl.AssemblyResult(ctx)
        for _ in range(2):
            fl.assemble_system(cfg.mesh, cfg.f, g, coef=cfg.coef, ctx=ctx, result=r)
            r.sizes()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            fl.assemble_system(cfg.mesh, cfg.f, g, coef=cfg.coef, ctx=ctx, result=r)
            r.sizes()
            ts.append(time.perf_counter() - t0)
        out[f"{name}_g={g}"] = round(1e3 * float(np.median(ts)), 3)
print(json.dumps(out))
