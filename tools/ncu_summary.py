"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"][: int(sys.argv[2]) if len(sys.argv) > 2 else 90]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e3:10.1f} {v[1] / 1e3 / v[0]:9.2f} {100 * v[1] / tot:5.1f}%  {k}")
print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
