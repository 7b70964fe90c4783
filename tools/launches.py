"""Summarise an ncu launch-list CSV (gpu__time_duration.sum): per kernel name,
count and mean microseconds over the last N launches."""
import csv
import sys
from collections import defaultdict

f = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
rows = list(csv.reader(l for l in open(f) if not l.startswith("==")))
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[vi]]
data = data[-last:]
agg = defaultdict(list)
for k, v in data:
    agg[k.split("(")[0][:70]].append(v)
for k, v in agg.items():
    print(f"{len(v):4d}  {sum(v)/len(v)/1e3:9.2f} us  {k}")
