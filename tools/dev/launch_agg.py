"""Aggregate an ncu launch list by kernel name (total us, count)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] in ("ns", "nsecond") else 1.0)
            k = d["Kernel Name"].split("(")[0][:60]
            agg[k][0] += v
            agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{us:10.1f} us  {n:4d}  {100 * us / tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
