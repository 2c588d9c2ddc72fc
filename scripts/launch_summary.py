"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
count and total time over the last `frac` of the launches."""
import collections
import csv
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h, data = None, []
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum":
            data.append(d)
n = len(data)
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data[int(n * (1 - frac)):]:
    k = d["Kernel Name"].split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"launches {n}, summarised {int(n * frac)}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v[1] / 1e3:10.1f} us {v[0]:6d}  {k}")
print(f"total {tot / 1e3:.1f} us")
