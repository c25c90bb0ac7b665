"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
mean device time and share of the listed time (cold-cache, serialised by ncu)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[i], rows[i + 1:]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
agg = defaultdict(list)
for r in data:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", ""))
        unit = r[unit_i] if unit_i is not None else "ns"
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | mean ms | share |")
print("|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {k} | {len(v)} | {sum(v) / len(v):.3f} | {100 * sum(v) / tot:.1f} % |")
