"""Markdown table of the bench lines under profiles/bench/bench_<tag>_*.json. Usage: python scripts/bench_table.py r02"""
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
print(f"# bench lines, tag `{tag}` (one B200 per run; `profiles/bench/bench_{tag}_*.json`)\n")
print("| line | schedule / objective | ms per step | tokens/s | roofline kernel | frac (of measured peak) | "
      "fwd frac | step frac | SM MHz (reasons) | cpu_baseline tokens/s (cores) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(root, "profiles", "bench", f"bench_{tag}_*.json"))):
    name = os.path.basename(f)[len(f"bench_{tag}_"):-5]
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    c = d.get("config") or {}
    r = d.get("roofline") or {}
    k = d.get("kernels") or {}
    cl = d.get("clocks") or {}
    cb = d.get("cpu_baseline") or {}
    sched = c.get("schedule") or c.get("objective") or d.get("impl", "")
    fr = r.get("frac")
    print(f"| {name} | {sched} | {d['ms_per_step']:.4g} | {d['value']:.4g} | {r.get('kernel', '—')} | "
          f"{'' if fr is None else f'{fr:.3f}'} | {k.get('fwd_frac', 0) and round(k['fwd_frac'], 3) or '—'} | "
          f"{k.get('step_frac', 0) and round(k['step_frac'], 3) or '—'} | {cl.get('sm_mhz')} ({','.join(cl.get('reasons') or [])}) | "
          f"{cb.get('value') and round(cb['value']) or '—'} ({cb.get('cores', '—')}) |")
