"""Per-opcode and per-source-line totals of an ncu SASS source export.

usage: sass_prof.py <sass.csv> <lib.so> <mangled kernel name> <n_units> [outer-file] [top]

Prints executed warp instructions, shared-memory wavefronts, global tag requests
and stall samples per unit (e.g. per column), by opcode and by source line of
`outer-file` (inlined code is charged to the line it was inlined at).
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

sass_csv, lib, kname, n_units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
outer = sys.argv[5] if len(sys.argv) > 5 else None
top = int(sys.argv[6]) if len(sys.argv) > 6 else 40
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
KEYS = {'inst': 'Instructions Executed', 'thr': 'Thread Instructions Executed',
        'smp': 'Warp Stall Sampling (All Samples)', 'wsh': 'L1 Wavefronts Shared',
        'tagg': 'L1 Tag Requests Global', 'l2s': 'L2 Theoretical Sectors Global'}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    d = {k: int(r[ix[h]] or 0) for k, h in KEYS.items()}
    d['addr'] = int(r[0], 16)
    d['src'] = r[1].strip()
    recs.append(d)
base = recs[0]['addr']
tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for f in os.listdir(tmp):
    if not f.endswith('.cubin'):
        continue
    txt = subprocess.run(['nvdisasm', '-gi', os.path.join(tmp, f)], capture_output=True, text=True).stdout
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
tot = {k: sum(r[k] for r in recs) for k in KEYS}
print('per unit:', {k: round(v / n_units, 2) for k, v in tot.items()})
oc = {k: Counter() for k in KEYS}
lc = {k: Counter() for k in KEYS}
for r in recs:
    s = r['src'].split()
    op = (s[1] if s[0].startswith('@') else s[0]).split('.')[0]
    ln = line_of.get(r['addr'] - base, ('?', 0))
    for k in KEYS:
        oc[k][op] += r[k]
        lc[k][ln] += r[k]
print('opcode          inst/u   thr/inst  shared-wf/u  gl-tags/u  samples%')
for op, v in oc['inst'].most_common(top):
    print(f'  {op:12s} {v / n_units:8.2f} {oc["thr"][op] / max(v, 1):8.1f} {oc["wsh"][op] / n_units:10.2f} '
          f'{oc["tagg"][op] / n_units:10.2f} {100 * oc["smp"][op] / tot["smp"]:8.1f}')
print('line                      inst/u   thr/inst  shared-wf/u  gl-tags/u  samples%')
for ln in sorted(lc['inst'], key=lambda k: (k[0] != outer, k[1])):
    v = lc['inst'][ln]
    if v / n_units < 0.5:
        continue
    print(f'  {ln[0]:>16s}:{ln[1]:<5d} {v / n_units:8.2f} {lc["thr"][ln] / max(v, 1):8.1f} {lc["wsh"][ln] / n_units:10.2f} '
          f'{lc["tagg"][ln] / n_units:10.2f} {100 * lc["smp"][ln] / tot["smp"]:8.1f}')
