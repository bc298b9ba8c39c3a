"""One write_matrix_market of an assembled config on the device (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib, configs  # noqa: E402

cfg = configs.build(sys.argv[1] if len(sys.argv) > 1 else "C4")
ctx = fl.Context.default()
r = fl.AssemblyResult(ctx)
fl.run(cfg.mesh, _lib.OUT_STIFFNESS, coef=cfg.coef, ctx=ctx, result=r)
t = fl.Text(ctx)
print(len(fl.write_result_matrix_market(r, text=t)))
