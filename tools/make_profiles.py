"""Write profiles/ summaries from gpurun_out/ ncu exports.

  python tools/make_profiles.py <round-tag> CONFIG...
reads gpurun_out/ll_<cfg>.csv (launch lists: gpu__time_duration.sum +
dram bytes per kernel, one assemble_system step, ncu --clock-control none)
and writes profiles/<tag>_launches_<cfg>.txt plus profiles/traffic.json
(dram bytes of the whole step and of the column kernel k_columns4, read by
bench.py as roofline.traffic / roofline.dominant_kernel.traffic).
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOMINANT = "k_columns4"
tag = sys.argv[1]
traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for c in sys.argv[2:]:
    rows = [r for r in csv.reader(open(os.path.join(ROOT, "gpurun_out", f"ll_{c}.csv"))) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        d[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    # tools/one_step.py runs a warm-up assembly first: keep the last step only
    # (from its first plan kernel, k4_bbox, on)
    starts = [i for (i, k) in sorted(d) if k.startswith("k4_bbox")]
    if starts:
        d = {ik: m for ik, m in d.items() if ik[0] >= starts[-1]}
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in d.values())
    lines = [f"# {c}: one steady-state step, fl_assemble(FL_OUT_SYSTEM | FL_REPLAN), ncu --clock-control none,",
             "# serialized cold-cache launches; time share is what matters, not the absolute",
             f"{'id':>3} {'kernel':60s} {'time_us':>10} {'share':>6} {'dram_rd_MB':>11} {'dram_wr_MB':>11}"]
    step_bytes, kern_bytes, kern_t = 0.0, 0.0, 0.0
    for (i, k), m in sorted(d.items()):
        t = m.get("gpu__time_duration.sum", 0)
        rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        lines.append(f"{i:3d} {k[:60]:60s} {t/1e3:10.1f} {100*t/tot:5.1f}% {rd/1e6:11.1f} {wr/1e6:11.1f}")
        step_bytes += rd + wr
        if DOMINANT in k:
            kern_bytes += rd + wr
            kern_t += t
    lines.append(f"# total {tot/1e6:.3f} ms, dram {step_bytes/1e9:.3f} GB; {DOMINANT} {kern_t/1e6:.3f} ms "
                 f"({100*kern_t/max(tot,1):.1f}%), dram {kern_bytes/1e9:.3f} GB")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches_{c}.txt"), "w").write("\n".join(lines) + "\n")
    traffic[c] = {"step_dram_bytes": step_bytes, "kernel_dram_bytes": kern_bytes,
                  "source": f"profiles/{tag}_launches_{c}.txt (ncu dram__bytes_read.sum+write.sum per step)"}
    print("\n".join(lines[-3:]))
json.dump(traffic, open(traffic_path, "w"), indent=1)
