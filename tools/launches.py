"""Summarise an ncu launch-list CSV: per kernel name, count and mean duration
over the last N launches, plus mean DRAM bytes read / written per launch when
the list carries dram__bytes_read.sum / dram__bytes_write.sum.

  python tools/launches.py gpurun_out/launches.csv [N]
"""
import csv
import sys
from collections import defaultdict

f = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
rows = list(csv.reader(l for l in open(f) if not l.startswith("==")))
hdr = rows[0]
ii, ki, mi, ui, vi = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launch = {}  # launch id -> (kernel, {metric: value in us / bytes})
for r in rows[1:]:
    if not r[vi]:
        continue
    k, m = launch.setdefault(r[ii], (r[ki], {}))
    m[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
ids = sorted(launch, key=int)[-last:]
agg = defaultdict(list)
for i in ids:
    k, m = launch[i]
    agg[k.split("(")[0][:70]].append(m)
for k, ms in agg.items():
    mean = lambda key: sum(m.get(key, 0.0) for m in ms) / len(ms)  # noqa: E731
    line = f"{len(ms):4d}  {mean('gpu__time_duration.sum'):9.2f} us"
    if any("dram__bytes_read.sum" in m for m in ms):
        line += f"  read {mean('dram__bytes_read.sum'):12.0f} B  write {mean('dram__bytes_write.sum'):10.0f} B"
    print(f"{line}  {k}")
