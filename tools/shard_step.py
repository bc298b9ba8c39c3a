"""Time ONE rank's share of a sharded step on one GPU (no other rank runs).

usage: shard_step.py CONFIG WORLD [RANK ...]   ->  one JSON line per rank

A rank's step needs nothing from the other ranks until the count exchange, so
its device time can be measured alone: the step of a G-GPU run is the max over
ranks of these numbers plus one 32-byte all_gather.  (This is a projection from
single-GPU measurements, not a multi-GPU measurement.)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FL_PROFILE", "1")
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib, configs  # noqa: E402
from paper_1804_05156_b200.shard import ShardedAssembler  # noqa: E402

name, world = sys.argv[1], int(sys.argv[2])
ranks = [int(x) for x in sys.argv[3:]] or [0]
cfg = configs.build(name)
ctx = fl.Context.default()
for rank in ranks:
    sa = ShardedAssembler(cfg.mesh, rank, world, ctx=ctx)
    res = fl.AssemblyResult(ctx)
    what = _lib.OUT_SYSTEM | _lib.REPLAN
    ms, ph = [], []  # the library's own CUDA events around plan / partition / numeric phases
    for k in range(8):
        sa.assemble(what, f=cfg.f, coef=cfg.coef, g_dirichlet=0.0, result=res)
        res.sizes()
        t = ctx.last_timings()
        if k >= 3:
            ms.append(sum(t[:3]))
            ph.append(t)
    s = res.sizes()
    print(json.dumps({"config": name, "world": world, "rank": rank, "cols": s.n, "nnz": s.nnz,
                      "ms_per_step": float(np.mean(ms)),
                      "phases_ms": {"plan": float(np.mean([p[0] for p in ph])),
                                    "partition": float(np.mean([p[1] for p in ph])),
                                    "numeric": float(np.mean([p[2] for p in ph]))},
                      "v4": os.environ.get("FL_V4", "1")}))
    del sa, res
