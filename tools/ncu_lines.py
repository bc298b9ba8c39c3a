"""Map an ncu SASS source export onto CUDA source lines via nvdisasm -g line info.

usage: ncu_lines.py <sass.csv> <lib.so> <mangled kernel name> [top] [outer-file]

With outer-file (e.g. fl_columns3.cu), inlined code is charged to the line of
that file it was inlined at, and a phase table is printed for PHASES below.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

sass_csv, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
outer = sys.argv[5] if len(sys.argv) > 5 else None
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, ii, si = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
recs = [(int(r[ia], 16), int(r[ii] or 0), int(r[si] or 0)) for r in rows[2:] if len(r) >= len(hdr)]
base = recs[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for f in os.listdir(tmp):
    if not f.endswith('.cubin'):
        continue
    txt = subprocess.run(['nvdisasm', '-gi' if outer else '-g', os.path.join(tmp, f)],
                         capture_output=True, text=True).stdout
    i = txt.find('.text.' + kname + ':')
    if i < 0:
        continue
    seg = txt[i:]
    j = seg.find('.section', 100)
    seg = seg[:j if j > 0 else None]
    cur = None
    for l in seg.split('\n'):
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            if outer:
                for fm in re.finditer(r'"([^"]+)", line (\d+)', l):
                    if os.path.basename(fm.group(1)) == outer:
                        cur = (outer, int(fm.group(2)))
        m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
        if m2 and cur:
            line_of[int(m2.group(1), 16)] = cur
    break
exe, smp = Counter(), Counter()
for a, i, s in recs:
    k = line_of.get(a - base, ('?', 0))
    exe[k] += i
    smp[k] += s
ti, ts = sum(exe.values()), sum(smp.values())
print(f"total inst {ti:.3e}, samples {ts}")
for k, v in exe.most_common(top):
    print(f"exec {100*v/ti:5.1f}%  samp {100*smp[k]/ts:5.1f}%  {k[0]}:{k[1]}")
