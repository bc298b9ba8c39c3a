"""The reference's own CPU path (oracle/_ref, 1 thread) on the FULL C5 mesh, beside
the same path on the bench's bounded sample (unit_cube:64, same recipe), so the
per-element rate the reference arm reports from the sample can be checked
against the full size.  Prints one JSON line.

  python tools/ref_full_c5.py [--skip-full]

Test/measurement infrastructure (it calls oracle/_ref); never part of the product.
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_1804_05156_b200 import configs  # noqa: E402


def rss_gb():
    try:
        for line in open("/proc/self/status"):
            if line.startswith("VmHWM"):
                return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return None


def run(n):
    t0 = time.time()
    cfg = configs.build("C5", n=n)
    m = cfg.mesh
    coef = po.coefficient_c5(m.dim, m.nodes, m.elems)
    build_s = time.time() - t0
    secs, nnz, nnz_ff = po.ref_time_system(m.dim, m.nodes, m.elems, m.bd_flags, po.FIELD_CONST, 1.0, coef,
                                           reps=1)
    s = float(secs[0])
    return {"n": n, "n_elems": m.num_elems(), "n_nodes": m.num_nodes(), "nnz": int(nnz), "nnz_ff": int(nnz_ff),
            "seconds": s, "elements_per_s": m.num_elems() / s, "mesh_build_s": build_s}


def main():
    out = {"what": "femlite partition_boundary + assemble_blockwise(+coefficient) + assemble_load + "
                   "apply_neumann + apply_dirichlet + submatrix + b_f (oracle/_ref ref_time_system), 1 thread",
           "host": platform.node(), "cpu": platform.processor() or platform.machine(),
           "threads": 1}
    try:
        out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    out["sample"] = run(64)
    if "--skip-full" not in sys.argv:
        out["full"] = run(256)
        out["full_over_sample_rate"] = out["full"]["elements_per_s"] / out["sample"]["elements_per_s"]
    out["peak_rss_gb"] = rss_gb()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
