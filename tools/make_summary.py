"""profiles/<tag>_summary.md from gpurun_out/f_<cfg>.json bench lines (+ f_ref.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rows = []
for c in ["C1", "C2", "C3", "C4", "C5"]:
    p = os.path.join(ROOT, "gpurun_out", f"f_{c}.json")
    if not os.path.exists(p):
        continue
    d = json.loads(open(p).read().strip().splitlines()[-1])
    rows.append((c, d))
out = [f"# {tag}: bench.py results on one B200 (N=1)", "",
       "Each line: `python bench.py --config Cx` (defaults: 10 timed steps after 3 warm-up;"
       " step = plan + partition + stiffness + load + Dirichlet lift + A(free,free) + b_f)."
       " Device numbers are CUDA-event times with inputs resident in HBM; e2e is wall clock"
       " through the C-ABI from pinned host memory (3-deep pipeline of contexts); cpu = the"
       " reference's own CPU path (oracle/_ref, 1 thread) on the config's bounded sample.", "",
       "| cfg | workload | NT | ms/step | Gelem/s | e2e Gelem/s | cpu Melem/s | e2e / cpu | numeric-phase GB/s (frac of 6547.8) | plan / partition / records / column kernel / placement ms | clocks |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for c, d in rows:
    ph = d["phases_ms"]
    cpu = d.get("cpu_baseline")
    cpu_v = cpu["value"] / 1e6 if cpu else None
    e2e = d["e2e"]["value"] / 1e9 if d.get("e2e") else None
    ratio = f"{d['e2e']['value'] / cpu['value']:.0f}x" if cpu and d.get("e2e") else "-"
    out.append(f"| {c} | {d['config']['workload']} | {d['config']['n_elems']:,} | {d['ms_per_step']:.3f} | "
               f"{d['value'] / 1e9:.3f} | {e2e:.3f} | {cpu_v:.3f} | {ratio} | "
               f"{d['roofline']['achieved']:.0f} ({d['roofline']['frac']:.3f}) | "
               f"{ph['plan']:.3f} / {ph['partition']:.3f} / {ph['element_records']:.3f} / "
               f"{ph['column_kernel']:.3f} / {ph['placement']:.3f} | "
               f"{d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |"
               if cpu_v is not None and e2e is not None else
               f"| {c} | {d['config']['workload']} | {d['config']['n_elems']:,} | {d['ms_per_step']:.3f} | "
               f"{d['value'] / 1e9:.3f} | {e2e} | - | - | {d['roofline']['achieved']:.0f} "
               f"({d['roofline']['frac']:.3f}) | {ph['plan']:.3f} / {ph['partition']:.3f} / "
               f"{ph['element_records']:.3f} / {ph['column_kernel']:.3f} / {ph['placement']:.3f} | "
               f"{d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |")
p = os.path.join(ROOT, "gpurun_out", "f_ref.json")
if os.path.exists(p):
    d = json.loads(open(p).read().strip().splitlines()[-1])
    out += ["", f"`bench.py --impl reference`: {d['value'] / 1e6:.3f} Melem/s, {d['ms_per_step']:.1f} ms per "
            f"sample step ({d['cpu_baseline']['sample']})."]
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
