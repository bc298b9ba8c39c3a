"""Aggregate an ncu SASS source export by instruction-index region and stall reason."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
ii = hdr.index('Instructions Executed'); ti = hdr.index('Thread Instructions Executed')
si = hdr.index('Warp Stall Sampling (All Samples)')
agg = {}
tot_s = tot_i = 0
for n, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    b = n // W
    a = agg.setdefault(b, {'i': 0, 't': 0, 's': 0, 'r': {}, 'first': r[1].strip()[:40]})
    i = int(r[ii] or 0); s = int(r[si] or 0)
    a['i'] += i; a['t'] += int(r[ti] or 0); a['s'] += s
    tot_i += i; tot_s += s
    for k in reasons:
        v = int(r[hdr.index(k)] or 0)
        a['r'][k] = a['r'].get(k, 0) + v
print('total inst', tot_i, 'samples', tot_s)
for b, a in sorted(agg.items()):
    if a['s'] / tot_s < 0.01 and a['i'] / tot_i < 0.01:
        continue
    top = sorted(a['r'].items(), key=lambda x: -x[1])[:4]
    tops = ' '.join(f"{k[6:]}:{100*v/max(a['s'],1):.0f}%" for k, v in top)
    print(f"{b*W:5d}: exec {100*a['i']/tot_i:5.1f}% thr {a['t']/max(a['i'],1):4.1f} samp {100*a['s']/tot_s:5.1f}%  [{tops}]  {a['first']}")
