"""Aggregate ncu warp-stall samples per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hk = next(k for k, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hk]
iall = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float), ""])
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= iall or not r[0] or not r[0].isdigit():
        continue  # per-line rows carry the aggregated metrics
    a = agg[(fname[:10] + ":" + r[0], r[1].strip()[:64])]
    a[0] += num(r[iall])
    a[1] += num(r[iex])
    for i in stall:
        a[2][hdr[i][6:]] += num(r[i])
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot:.0f}")
for (ln, src), (s, ex, st, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{k}:{100 * v / max(s, 1):.0f}%" for k, v in reasons)
    print(f"{ln:>16s} {100 * s / tot:5.1f}% ex={ex:10.0f} {src:64s} {rs}")
