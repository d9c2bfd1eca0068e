"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel-name count / total / mean microseconds, sorted by total."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0][:70]
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "nsecond"
        us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000)
        agg[name].append(us)
tot = sum(sum(v) for v in agg.values())
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.1f} us {100 * sum(v) / tot:5.1f}%  n={len(v):4d}  mean={sum(v) / len(v):8.2f}  {name}")
print(f"{tot:10.1f} us total")
