"""Summarise an ncu report: key raw metrics + SASS opcode / stall histogram.
Usage: python tools/ncu_sass_hot.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for i, k in enumerate(h):
    if k in want or ("average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")):
        try:
            if float(v[i]) < 0.05:
                continue
        except ValueError:
            pass
        print(k, v[i])
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
r = list(csv.reader(io.StringIO(sass)))
hdr = r[1]
rows = [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]
ie, st = "Instructions Executed", "Warp Stall Sampling (All Samples)"
tot = sum(int(d[ie]) for d in rows)
tst = sum(int(d[st]) for d in rows)
print("total inst", tot, "stall samples", tst)
op, sst = collections.Counter(), collections.Counter()
for d in rows:
    t = d["Source"].split()
    o = t[1] if t[0].startswith("@") else t[0]
    op[o] += int(d[ie])
    sst[o] += int(d[st])
print("opcode  inst  %inst  stall%")
for o, c in sst.most_common(top):
    print(f"{o:28s} {op[o]:10d} {100 * op[o] / tot:5.1f} {100 * c / tst:5.1f}")
