"""Run a few assemble_system steps of one config (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = configs.build(name)
ctx = fl.Context.default()
r = fl.AssemblyResult(ctx)
for _ in range(steps):
    fl.assemble_system(cfg.mesh, cfg.f, 0.0, coef=cfg.coef, ctx=ctx, result=r)
    r.sizes()
print("ok", name, r.sizes().nnz)
