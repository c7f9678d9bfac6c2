"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per kernel name,
launches, mean / total us and share of the total."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[hdr.index("Kernel Name")].split("(")[0]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        d.setdefault(k, []).append(v)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):5d} mean={sum(v) / len(v):9.2f} us total={sum(v) / 1e3:9.3f} ms share={sum(v) / tot:6.3f}")
