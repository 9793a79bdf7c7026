"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.
Usage: python tools/launch_table.py launches.csv [top]"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr, agg, total, n = None, collections.defaultdict(lambda: [0, 0.0]), 0.0, 0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(ttr::.*|\(unnamed.*", "", d["Kernel Name"]).replace("ttr::<unnamed>::", "")[:80]
        us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
        total += us
        n += 1
    print(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{c:8d} {t:10.1f} {t / c:9.2f} {100 * t / total:5.1f}%  {name}")
    print(f"total {total:.1f} us over {n} launches")


if __name__ == "__main__":
    main()
