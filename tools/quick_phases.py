"""Device phases of one config (FL_PROFILE=1), for quick A/B runs: python tools/quick_phases.py C5 [steps]"""
import json
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = sys.argv[2] if len(sys.argv) > 2 else "5"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", cfg, "--no-e2e",
                      "--no-cpu-baseline", "--steps", steps], capture_output=True, text=True)
d = json.loads(out.stdout.strip().splitlines()[-1])
print(cfg, os.environ.get("TAG", ""), round(d["ms_per_step"], 3), "ms",
      {k: round(v, 3) for k, v in d["phases_ms"].items()}, "frac", round(d["roofline"]["frac"], 4),
      out.stderr.strip().splitlines()[-1:] if "L2" in out.stderr else "")
