"""BASELINE.md section 5 rows from the committed profiles (bench lines, reference arm, TT-SVD timing).
Usage: python tools/baseline_table.py [tag]   (tag = profiles prefix, default r02f)"""
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 2 - 1 and len(sys.argv) > 1 else "r02f"
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def load(name):
    p = os.path.join(root, name)
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def ms(x):
    return "—" if x is None else (f"{x:,.0f}" if x >= 100 else f"{x:.3g}")


rows = []
for cfg, label in [("1", "1"), ("2", "2"), ("3", "3 (KRP)"), ("4", "4"), ("5a", "5a"), ("5b", "5b")]:
    b = load(f"{tag}_bench{cfg}.json")
    one = load(f"{tag}_ref{cfg}_1thread.json")
    allc = load(f"{tag}_ref{cfg}.json")
    cb = b["cpu_baseline"]
    cpu_all_ms = allc["ms_per_step"] if allc else cb.get("ms_per_round", cb.get("seconds", 0) * 1e3 if cb.get("seconds") else None)
    cores = (allc or {}).get("cpu_baseline", {}).get("cores", cb["cores"])
    note = "" if allc or cfg != "5a" else " (128 of 4096 tensors)"
    r = b["roofline"]
    par = b["config"].get("parity") or ("ranks identical" if b["config"].get("ranks_identical", True) else "")
    rows.append(f"| {label} | {ms(one['ms_per_step']) if one else '—'} | {ms(cpu_all_ms)}{note}, {cores} | {b['ms_per_step']:.3g} | — | — | — | "
                f"{b.get('tflops_fp64', b['value']):.3g} | {r['frac']:.3f} of {r['bound']} peak ({r['kernel'].split(' ')[0][:40]}) | "
                f"≤ 1e-10, identical ranks (tests/test_gpu_parity.py full-size parity) |")
d3 = load(f"{tag}_det3.json")
d3c = load(f"{tag}_det3_cpu.json")
rows.insert(3, f"| 3 (TT-SVD) | — | {ms(d3c['cpu_s'] * 1e3) if d3c else '—'}, {d3c['cpu_threads'] if d3c else ''} | {d3['gpu_ms']:.3g} | — | — | — | "
               f"{d3['gpu_tflops']:.3g} | latency-bound (one-cluster Jacobi SVD) | ≤ 1e-10, identical ranks (`[3-det]`) |")
print("\n".join(rows))
