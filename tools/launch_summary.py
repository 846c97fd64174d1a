"""Summarise an ncu launch list (gpu__time_duration per launch) for the last
FMM step in it: per-kernel totals and shares."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, idi = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
ks = [(int(r[idi]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
names = [k[1] for k in ks]
last = max(i for i, n in enumerate(names) if "ingest_bounds" in n)
step = [s for s in ks[last:] if "probe" not in s[1]]
tot = sum(s[2] for s in step)
agg = collections.OrderedDict()
for _, n, v in step:
    key = n.split("(")[0].replace("void ", "")
    agg.setdefault(key, [0, 0])
    agg[key][0] += v
    agg[key][1] += 1
print(f"step: {len(step)} launches, {tot / 1e6:.3f} ms of kernel time (ncu, serialised, cold cache)")
for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v / 1e3:10.1f} us {c:4d}  {100 * v / tot:5.1f}%  {k[:100]}")
