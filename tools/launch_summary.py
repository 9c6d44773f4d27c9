"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    if len(r) > vi:
        d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/1e6:10.3f} ms {100*sum(v)/tot:5.1f}%  n={len(v):4d}  avg={sum(v)/len(v)/1e3:10.1f} us  {k}")
