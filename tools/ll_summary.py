"""Summarise gpurun_out/ll_<cfg>.csv launch lists (per-kernel time and DRAM bytes)."""
import collections
import csv
import sys

for c in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/ll_{c}.csv")) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        d[(int(r[ii]), r[ki][:40])][r[mi]] = float(r[vi].replace(",", ""))
    starts = [i for (i, k) in sorted(d) if k.startswith("k4_bbox")]
    if starts:  # the last (steady-state) step only
        d = {ik: m for ik, m in d.items() if ik[0] >= starts[-1]}
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in d.values()) / 1e6
    print(c, f"total {tot:.3f} ms over {len(d)} launches")
    for (i, k), m in sorted(d.items()):
        t = m.get("gpu__time_duration.sum", 0)
        if t > 50000:
            print(f"  {k:40s} {t/1e6:8.3f} ms  rd {m.get('dram__bytes_read.sum',0)/1e9:6.2f} GB"
                  f"  wr {m.get('dram__bytes_write.sum',0)/1e9:6.2f} GB")
