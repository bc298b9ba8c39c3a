"""Summarise one ncu --set full report (key counters, stall mix, source-line
instruction shares) into a text file under profiles/.

  python tools/ncu_summary.py <report.ncu-rep> <out.txt> <title> [mangled-kernel] [outer-file]
"""
import csv
import io
import os
import subprocess
import sys

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
kname = sys.argv[4] if len(sys.argv) > 4 else None
outer = sys.argv[5] if len(sys.argv) > 5 else None
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
lines = [f"# {title}", f"# ncu --set full --import-source on --clock-control none ({os.path.basename(rep)})", ""]
for w in want:
    if w in h:
        i = h.index(w)
        lines.append(f"{w:70s} {v[i][:60]:>16s} {u[i]}")
st = [(h[i], v[i]) for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
tot = sum(float(x) for _, x in st if x.replace(".", "", 1).isdigit())
lines += ["", "# warp-state samples (share of stall samples)"]
for n, x in sorted(st, key=lambda a: -float(a[1]) if a[1].replace(".", "", 1).isdigit() else 0)[:8]:
    lines.append(f"{n:70s} {100 * float(x) / tot:5.1f}%")
if kname:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    tmp = "/tmp/_ncu_src.csv"
    open(tmp, "w").write(src)
    args = [sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp,
            os.path.join(ROOT, "paper_1804_05156_b200", "libfemlite_b200.so"), kname, "25"]
    if outer:
        args.append(outer)
    res = subprocess.run(args, capture_output=True, text=True).stdout
    lines += ["", "# executed instructions / stall samples by source line (tools/ncu_lines.py)"] + res.splitlines()
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:30]))
