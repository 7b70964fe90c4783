"""Top SASS lines by warp-stall samples from an ncu report (--page source)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia][-5:], r[isrc].strip()) for r in rows[1:] if len(r) > iss]
tot = sum(d[0] for d in data)
print("total samples", tot)
for i, d in enumerate(data):
    pass
order = sorted(range(len(data)), key=lambda i: -data[i][0])[:top]
for i in sorted(order):
    s, a, src = data[i]
    print(f"{s:7d} {100*s/tot:5.1f}%  {a}  {src[:90]}")
