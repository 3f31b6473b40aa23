"""Launch-list table from `ncu --metrics gpu__time_duration.sum --csv --log-file x.csv <cmd>`:
launches, mean and total device time and share per kernel (cold-cache, serialised: compare shares).
usage: python tools/ncu_launches.py launches.csv [header lines...] > profiles/<name>.txt"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr_i]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr_i + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0]
        agg[name].append(float(r[vi].replace(",", "")) / (1e3 if "ns" in (r[h.index("Metric Unit")] if "Metric Unit" in h else "") else 1.0))
tot = sum(sum(v) for v in agg.values())
for line in sys.argv[2:]:
    print("# " + line)
print("# launches  mean_us  total_us  share  kernel")
for name, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):9d} {sum(v) / len(v):8.1f} {sum(v):9.1f} {100 * sum(v) / tot:5.1f}%  {name}")
