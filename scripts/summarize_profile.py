#!/usr/bin/env python
"""Summarise a gpurun profiling session into profiles/<tag>/summary.md.

    python scripts/summarize_profile.py <tag> [<outdir> <label> <bench.json>]

Reads gpurun_out/<tag>_launches.csv (ncu --metrics gpu__time_duration.sum launch list)
and gpurun_out/<tag>_adjoint.ncu-rep (ncu --set full of the adjoint), writes the
per-kernel shares of device time, the adjoint's DRAM bytes per launch, and the top
stall reasons; also updates profiles/adjoint_traffic.json (read by bench.py).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip()
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def ncu_raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    tag = sys.argv[1]
    outdir = os.path.join(ROOT, "profiles", sys.argv[2] if len(sys.argv) > 2 else tag)
    label = sys.argv[3] if len(sys.argv) > 3 else "summary"
    os.makedirs(outdir, exist_ok=True)
    g = os.path.join(ROOT, "gpurun_out")
    lines = [f"# Profile summary {tag}", ""]
    bench = sys.argv[4] if len(sys.argv) > 4 else os.path.join(g, f"{tag}_bench.json")
    b = None
    if os.path.exists(bench):
        try:
            b = json.loads(open(bench).read().strip().splitlines()[-1])
            lines += ["## bench line", "", "```", json.dumps({k: b[k] for k in ("value", "unit", "ms_per_step", "roofline", "hbm", "clocks") if k in b}, indent=1), "```", ""]
        except Exception as e:  # noqa: BLE001
            lines += [f"(bench json unreadable: {e})", ""]
    lp = os.path.join(g, f"{tag}_launches.csv")
    if os.path.exists(lp):
        tot, cnt = launch_shares(lp)
        T = sum(tot.values())
        lines += ["## launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache serialised: compare shares)", "",
                  "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
        for k in sorted(tot, key=lambda k: -tot[k]):
            lines.append(f"| {k} | {cnt[k]} | {tot[k] / 1e6:.3f} | {tot[k] / cnt[k] / 1e3:.2f} | {tot[k] / T:.3f} |")
        lines.append("")
    rp = os.path.join(g, f"{tag}_adjoint.ncu-rep")
    if os.path.exists(rp):
        hdr, units, data = ncu_raw(rp)
        want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
        lines += ["## ncu --set full, adjoint kernel", ""]
        traffic = {}
        for row in data:
            d = dict(zip(hdr, row))
            u = dict(zip(hdr, units))
            for w in want:
                if w in d:
                    lines.append(f"- {w}: {d[w]} {u.get(w, '')}")
            stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for h, v in d.items()
                      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                      and v.replace(".", "", 1).isdigit()]
            stalls.sort(key=lambda x: -x[1])
            tot = sum(v for _, v in stalls) or 1.0
            lines.append("- top stall reasons (pc samples): " + ", ".join(f"{n} {v / tot:.0%}" for n, v in stalls[:6]))
            lines.append("")

            def to_bytes(key):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(key, "byte"), 1)
                return float(d[key].replace(",", "")) * mult
            if "dram__bytes_read.sum" in d:
                traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
        if b is not None and traffic:
            key = f"{b['config']['workload'].split(':')[0]}:b{b['config']['b_phi']}:gpus{b['n_gpus']}:v{b['config'].get('adjoint_variant', 0)}"
            tp = os.path.join(ROOT, "profiles", "adjoint_traffic.json")
            dd = json.load(open(tp)) if os.path.exists(tp) else {}
            dd[key] = traffic
            json.dump(dd, open(tp, "w"), indent=1)
            lines.append(f"traffic per launch (dram read+write): {traffic:.4g} B -> profiles/adjoint_traffic.json[{key}]")
    open(os.path.join(outdir, f"{label}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
