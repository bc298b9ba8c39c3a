"""One warm-up assembly (synchronous first plan), then `steps` steady-state
steps -- fl_assemble(FL_OUT_SYSTEM | FL_REPLAN), the bench's step -- of one config
(for ncu captures: the LAST step is the one to read)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib, api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = configs.build(name)
ctx = fl.Context.default()
r = fl.AssemblyResult(ctx)
fl.assemble_system(cfg.mesh, cfg.f, 0.0, coef=cfg.coef, ctx=ctx, result=r)
r.sizes()
for _ in range(steps):
    api.run(cfg.mesh, _lib.OUT_SYSTEM | _lib.REPLAN, f=cfg.f, coef=cfg.coef, g_dirichlet=0.0, ctx=ctx, result=r)
    r.sizes()
print("ok", name, r.sizes().nnz)
