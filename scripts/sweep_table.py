#!/usr/bin/env python
"""Collect gpurun_out/<tag>_*.json bench lines into profiles/<round>/sweep_<tag>/ + README table.

    python scripts/sweep_table.py <tag> <round>
"""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "profiles", rnd, f"sweep_{tag}")
os.makedirs(out, exist_ok=True)
rows = ["| run | iter/s | ms/step | dominant kernel | achieved | frac of peak | e2e iter/s | oracle iter/s (cores) | SM MHz |",
        "|---|---|---|---|---|---|---|---|---|"]
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_*.json"))):
    name = os.path.basename(f)[len(tag) + 1:-5]
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    if "value" not in d:
        continue
    shutil.copy(f, os.path.join(out, os.path.basename(f)[len(tag) + 1:]))
    rf = d.get("roofline") or {}
    cb = d.get("cpu_baseline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    clk = d.get("clocks") or {}
    rows.append(f"| {name} | {d['value']:.4g} | {d.get('ms_per_step') or 0:.3f} | {str(rf.get('kernel', '-'))[:40]} | "
                f"{rf.get('achieved', 0):.1f} {rf.get('unit', '')} | {rf.get('frac', 0):.3f} | "
                f"{'-' if e2e is None else f'{e2e:.4g}'} | {cb.get('value', '-') if not cb else f'{cb[chr(118)+chr(97)+chr(108)+chr(117)+chr(101)]:.3g} ({cb.get(chr(99)+chr(111)+chr(114)+chr(101)+chr(115))})'} | "
                f"{clk.get('sm_mhz')} {' '.join(clk.get('reasons') or [])} |")
open(os.path.join(out, "README.md"), "w").write(f"# bench sweep {tag} (one B200, scripts/gpu_sweep.sh)\n\n" + "\n".join(rows) + "\n")
print("\n".join(rows))
