"""Per-phase cycle breakdown of the tiled column kernel (FL_PHASES=1)."""
import ctypes as C
import os
import sys
import time

os.environ["FL_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib, configs  # noqa: E402

names = ["keys", "geometry", "folds", "sort/drop", "look-back", "writes"]
for cfgname in sys.argv[1:] or ["C4"]:
    cfg = configs.build(cfgname, f_mode="samples")
    ctx = fl.Context.default()
    r = fl.AssemblyResult(ctx)
    for _ in range(3):
        fl.assemble_system(cfg.mesh, cfg.f, 0.0, coef=cfg.coef, ctx=ctx, result=r)
        r.sizes()
    out = (C.c_uint64 * 6)()
    _lib.check(_lib.lib().fl_phase_cycles(ctx.handle, out))
    tot = sum(out)
    t0 = time.perf_counter()
    fl.assemble_system(cfg.mesh, cfg.f, 0.0, coef=cfg.coef, ctx=ctx, result=r)
    r.sizes()
    dt = time.perf_counter() - t0
    print(cfgname, f"wall {dt*1e3:.2f} ms", " ".join(f"{n}:{100*v/tot:.1f}%" for n, v in zip(names, out)),
          f"total {tot:.3e} cycles")
