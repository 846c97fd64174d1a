"""Top SASS lines by stall samples from `ncu -i rep --page source --csv --print-source sass`:
    python tools/ncu_hot.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ia, isrc, iall, inot = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Warp Stall Sampling (Not-issued Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iall] or 0), int(r[inot] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, ns, a, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.2f}% {100 * ns / tot:5.2f}% {a} {src[:90]}")
