"""Extract the roofline-relevant metrics of the first kernel in an ncu report
into a small JSON summary (committed under profiles/ and read by bench.py).
Usage: python tools/ncu_to_json.py report.ncu-rep out.json [note]"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Tbyte": 1e12}

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
out = {"kernel": vals[hdr.index("Kernel Name")]}
for i, k in enumerate(hdr):
    if k in WANT:
        v = vals[i].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            out[WANT[k]] = v
            continue
        u = units[i]
        if WANT[k] == "duration":
            out["duration_s"] = x * SCALE.get(u, 1.0)
        elif WANT[k] in ("dram_read", "dram_write", "l2_bytes"):
            out[WANT[k] + "_bytes"] = x * SCALE.get(u, 1.0)
        else:
            out[WANT[k]] = x
if len(sys.argv) > 3:
    out["note"] = sys.argv[3]
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
