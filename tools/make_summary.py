"""profiles/<tag>_summary.md from bench lines.

  python tools/make_summary.py <tag> [prefix]     (default prefix: ev_)
reads gpurun_out/<prefix>bench_<cfg>.json, <prefix>ref.json and
<prefix>ref_full_c5.json (tools/runs/evidence.sh)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
pre = sys.argv[2] if len(sys.argv) > 2 else "ev_"


def load(name):
    p = os.path.join(ROOT, "gpurun_out", name)
    if not os.path.exists(p):
        return None
    lines = [l for l in open(p).read().strip().splitlines() if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


out = [f"# {tag}: bench.py on one B200 (N=1)", "",
       "`python bench.py --config Cx` (10 timed steps after 3 warm-up). Step = Morton labels + label "
       "plan rebuilt from the raw arrays + partition + FaceLists + stiffness + load + Dirichlet lift + "
       "A(free,free) + b_f (`fl_assemble(FL_OUT_SYSTEM|FL_REPLAN)`). Device numbers: CUDA events, inputs "
       "resident in HBM. `frac` = B_SL / step / measured HBM peak (SURVEY §8(d)). e2e: C-ABI from pinned "
       "host memory, 3-deep pipeline; e2e 1-call: one un-pipelined call. cpu: the reference's own path "
       "(oracle/_ref) on all host threads, bounded sample of the config family.", "",
       "| cfg | NT | ms/step | Gelem/s | frac (B_SL) | e2e Gelem/s | e2e 1-call ms | cpu Melem/s (threads) | "
       "labels+plan / partition+faces / xl+column / placement ms | column kernel ms (share) | clocks |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for c in ["C1", "C2", "C3", "C4", "C5"]:
    d = load(f"{pre}bench_{c}.json")
    if not d:
        continue
    ph = d["phases_ms"]
    cpu = d.get("cpu_baseline") or {}
    e2e = d.get("e2e") or {}
    single = d.get("e2e_single") or {}
    dk = d["roofline"].get("dominant_kernel", {})
    out.append(
        f"| {c} | {d['config']['n_elems']:,} | {d['ms_per_step']:.3f} | {d['value'] / 1e9:.3f} | "
        f"{d['roofline']['frac']:.4f} | {e2e.get('value', 0) / 1e9:.3f} | {single.get('ms', 0):.1f} | "
        f"{cpu.get('value', 0) / 1e6:.2f} ({cpu.get('cores', '-')}) | "
        f"{ph['plan']:.3f} / {ph['partition']:.3f} / {ph['numeric'] - ph['placement']:.3f} / {ph['placement']:.3f} | "
        f"{ph['column_kernel']:.3f} ({dk.get('share_of_step') or 0:.0%}) | "
        f"{d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |")
r = load(f"{pre}ref.json")
if r:
    out += ["", f"`bench.py --impl reference`: {r['value'] / 1e6:.3f} Melem/s, {r['ms_per_step']:.1f} ms per "
            f"sample round on {r['cpu_baseline']['cores']} threads ({r['cpu_baseline']['sample']})."]
f = load(f"{pre}ref_full_c5.json")
if f:
    s = f["sample"]
    line = (f"\nThe reference on one thread (`tools/ref_full_c5.py`, {f.get('cpu_model', '')}): sample "
            f"unit_cube:64 {s['elements_per_s'] / 1e6:.3f} Melem/s ({s['seconds']:.1f} s)")
    if "full" in f:
        g = f["full"]
        line += (f"; FULL C5 unit_cube:256 {g['elements_per_s'] / 1e6:.3f} Melem/s ({g['seconds']:.1f} s, "
                 f"peak RSS {f.get('peak_rss_gb') or 0:.1f} GB): full/sample per-element rate "
                 f"{f['full_over_sample_rate']:.2f}.")
    out.append(line)
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
