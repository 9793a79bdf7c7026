#!/usr/bin/env python3
"""bench.py — headline benchmark: fixed-rank KRP TT-rounding (BASELINE config 5b)
on B200 through the library's C ABI.

Workload (config 5b, BASELINE.json configs[4](b)): d=20, n=128, Y = X + 1e-8 Z
with X a unit-norm rank-300 Gaussian TT and Z a unit-norm rank-700 Gaussian TT
(formal ranks 1000, 18.4 GB of cores), rounded with round_fixed_krp(Y, {320}x19,
seed 7) — KRP sketch width l = 320. Cores are drawn on the device from Philox
(synthetic; the reference has no dataset for this path). A "step" is one full
round_fixed_krp call (sketch + left-to-right Rand-Orth sweep).

  value  = algorithmic fp64 TFLOP/s of the whole round (reference flop charges,
           proj/core/src/linalg.cpp:25-61) with the input resident in HBM,
           summed over ranks (N>1: every rank rounds its own independent 5b
           tensor — batch sharding, no collective; "scaling": "weak").
  e2e    = the same metric through the C ABI with host buffers: H2D upload of
           the input from pinned memory + rounding + D2H download of the result
           inside the timed region.
  roofline: the KRP sketch contraction kernel (krp_step = TMA-fed DMMA GEMM +
           split-K reduce) against the measured fp64 DMMA peak; traffic from
           the committed ncu capture of one launch at the same shape.
  cpu_baseline: the CPU oracle (restatement of the reference on its OpenBLAS/LAPACK
           backend, all host threads) on the FULL config: one round_fixed_krp of
           the same input (downloaded from the device), wall clock around the call.

--impl reference times that CPU implementation alone on the same config (input
rebuilt on the host: the Philox cores are bitwise the device's), one full round
per step (the reference itself cannot be built here: Eigen is absent — see
DESIGN.md §4).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading

import numpy as np
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KRP TT-rounding time (ms) and fp64 TFLOP/s vs peak at 1/2/4/8 B200 vs host CPU"
FP64_PEAK_TFLOPS = 36.9  # measured: DMMA m8n8k4 microbenchmark, profiles/r01_box_probe.log
PEAK_SOURCE = "measured fp64 DMMA (mma.sync m8n8k4) burst peak on this pool's B200, profiles/r01_box_probe.log"

CFG5B = dict(d=20, n=128, rx=300, rz=700, eps=1e-8, ell=320, seed=1005, round_seed=7)
CFG3 = dict(d=30, n=64, rx=100, rz=300, eps=1e-8, ell=110, seed=1003)
CFG1 = dict(d=10, n=20, rx=10, rz=40, eps=1e-4, ell=15, seed=1001)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="5b", choices=["5b", "1", "2", "3", "4", "5a"],
                    help="BASELINE config: 5b (default, the headline), 1 and 3 (fixed rank), 2 and 4 "
                         "(adaptive rank), 5a (batch of 4096 tensors)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0,
                    help="host threads of the CPU reference / cpu_baseline (default: all cores)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharding", default="tensor", choices=["tensor", "batch"],
                    help="N>1 on config 5b: ONE tensor over the N GPUs (default; column-sharded KRP sketch + "
                         "NCCL all-gather, row-sharded Rand-Orth sweep with an NVLink TSQR per mode; strong "
                         "scaling), or an independent tensor per rank (batch; weak scaling)")
    ap.add_argument("--local-ranks", type=int, default=0,
                    help="run the sharded driver with this many ranks simulated on ONE GPU (same code and "
                         "kernels as the NCCL run; a functional check, not a multi-GPU timing)")
    return ap.parse_args()


def maybe_spawn(args):
    """`bench.py --gpus N` (N > 1) started without a launcher re-executes itself under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference (the oracle restatement of the reference, on its OpenBLAS/LAPACK
# backend) on the FULL config — used by the cpu_baseline leg and --impl reference

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import py_oracle as O
    return O


def cpu_threads(args=None) -> int:
    if args is not None and getattr(args, "cpu_threads", 0):
        return args.cpu_threads
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_input(O, cfg):
    """The bench input rebuilt on the host: the Philox cores are bitwise the device's
    (oracle random_philox_tt == ttr_tt_random_philox), each part scaled to unit norm
    (sqrt(dot), a GEMM-only pass) and combined by formal_sum."""
    d, n = cfg["d"], cfg["n"]
    x = O.random_philox_tt([n] * d, [1] + [cfg["rx"]] * (d - 1) + [1], O.derive_seed(cfg["seed"], 1))
    x = O.scaled(x, 1.0 / math.sqrt(O.dot(x, x)))
    z = O.random_philox_tt([n] * d, [1] + [cfg["rz"]] * (d - 1) + [1], O.derive_seed(cfg["seed"], 2))
    z = O.scaled(z, cfg["eps"] / math.sqrt(O.dot(z, z)))
    return O.formal_sum([x, z])


def cpu_round(O, x, ranks, seed):
    """One round_fixed_krp on the host, wall clock around the call only
    (tools/ttround_main.cpp:156-160). Returns (seconds, charged flops)."""
    sec = C.c_double()
    fl = C.c_uint64()
    O._check(O.lib().ttro_time_round_fixed_krp(x._h, O._i64(ranks), C.c_int64(len(ranks)), C.c_uint64(seed),
                                               C.c_int(O.PHILOX), C.byref(sec), C.byref(fl)))
    return sec.value, fl.value


def cpu_desc(cfg, threads):
    return (f"the full config: round_fixed_krp(Y, {{{cfg['ell']}}}x{cfg['d'] - 1}, 7) on the same input "
            f"(d={cfg['d']}, n={cfg['n']}, ranks {cfg['rx']} + {cfg['eps']:g} x {cfg['rz']}), one round per step; "
            f"CPU oracle (restatement of the reference, OpenBLAS/LAPACK backend: dgemm, dgeqrf+dorgqr) on "
            f"{threads} host threads, wall clock around the call")


REF_BUDGET_S = 240.0  # CPU seconds of rounds the reference arm may spend (see run_reference)


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation of the path (the oracle
    port — the reference itself cannot be built here) on the host cores,
    on the same config, metric and unit as the GPU arm. Rank 0 only."""
    if rank != 0:
        return
    O = _oracle()
    threads = cpu_threads(args)
    O.set_backend("blas", threads)
    cfg = dict(CFG5B)
    if args.config == "3":
        cfg.update(CFG3)
    elif args.config == "1":
        cfg.update(CFG1)
    elif args.config != "5b":
        print(json.dumps({"impl": "reference", "unavailable": f"--impl reference covers configs 5b, 3 and 1 "
                                                                f"(asked: {args.config})"}), flush=True)
        return
    t0 = time.perf_counter()
    x = cpu_input(O, cfg)
    gen_s = time.perf_counter() - t0
    ranks = [cfg["ell"]] * (cfg["d"] - 1)
    # One step is one full round (16-17 s for 5b on 16 threads). The run is bounded
    # to REF_BUDGET_S of CPU rounds so that any --steps/--warmup ends within minutes:
    # at least one warm-up and two timed rounds, then as many of the asked ones as fit
    # (steps_run / warmup_run say what ran; the value is per round, so it is unaffected).
    t_run = time.perf_counter()
    first = cpu_round(O, x, ranks, 7)
    per = max(first[0], 1e-3)
    fit = max(3, int(REF_BUDGET_S / per))
    warm = min(args.warmup, max(1, fit - 2)) if args.warmup > 0 else 0
    steps = max(1, min(args.steps, fit - warm))
    for _ in range(max(0, warm - 1)):
        cpu_round(O, x, ranks, 7)
    res = ([] if warm > 0 else [first]) + [cpu_round(O, x, ranks, 7) for _ in range(steps - (0 if warm > 0 else 1))]
    secs = [r[0] for r in res]
    flops = res[0][1]
    ms = sum(secs) / len(secs) * 1e3
    tflops = flops / (ms * 1e-3) / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "steps_run": len(secs), "warmup_run": warm,
        "run_seconds": time.perf_counter() - t_run, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (host Philox Gaussian cores, bitwise the device generator)",
        "config": {"workload": f"config {args.config} fixed-rank KRP rounding round_fixed_krp(Y, "
                               f"{{{cfg['ell']}}}x{cfg['d'] - 1}, 7)", "d": cfg["d"], "n": cfg["n"],
                   "formal_rank": cfg["rx"] + cfg["rz"], "l": cfg["ell"], "same_config": True,
                   "flops_per_step": flops, "input_build_s": gen_s},
        "step_seconds": secs,
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": cpu_desc(cfg, threads)},
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML (pynvml,
    microseconds per query) when available, else nvidia-smi. (A spawned nvidia-smi
    stalls CUDA API calls for up to ~0.5 s, which host-driven adaptive rounds
    would feel; the NVML queries do not.)"""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, [reason flags in NAMES order])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((float(sm), float(mx), [bool(r & b) for b in bits]))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        vals = [v.strip() for v in out.stdout.strip().split(",")]
        if len(vals) == 6 and vals[0].replace(".", "").isdigit() and vals[1].replace(".", "").isdigit():
            self.samples.append((float(vals[0]), float(vals[1]), [v.lower() == "active" for v in vals[2:]]))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2][i]})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def build_input(P, ctx, cfg):
    d, n = cfg["d"], cfg["n"]
    from paper_2511_03598_b200.seeds import derive_seed
    rx = [1] + [cfg["rx"]] * (d - 1) + [1]
    rz = [1] + [cfg["rz"]] * (d - 1) + [1]
    x = P.TTTensor.random_philox([n] * d, rx, derive_seed(cfg["seed"], 1), ctx)
    z = P.TTTensor.random_philox([n] * d, rz, derive_seed(cfg["seed"], 2), ctx)
    x = P.scaled(x, 1.0 / P.norm_exact(x))
    z = P.scaled(z, cfg["eps"] / P.norm_exact(z))
    return P.formal_sum([x, z])


def run_ours(args, world, rank, local):
    import torch
    import paper_2511_03598_b200 as P
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    # a dedicated (non-default) stream: the library and the timing events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local, stream.cuda_stream)

    cfg = dict(CFG5B)
    if args.config == "3":
        cfg.update(CFG3)
    elif args.config == "1":
        cfg.update(CFG1)
    cfg["seed"] = cfg["seed"] + 1000 * rank  # independent tensor per rank
    y = build_input(P, ctx, cfg)
    ranks = [cfg["ell"]] * (cfg["d"] - 1)
    torch.cuda.synchronize()

    seed = cfg.get("round_seed", 7)

    def eager_step():
        return P.round_fixed_krp(y, ranks, seed)

    # flops per step (reference charges) and launch count, eager API
    ctx.reset_counters()
    l0 = ctx.kernel_launches()
    out = eager_step()
    torch.cuda.synchronize()
    flops = ctx.counters().total()
    sketch_flops = ctx.counters().sketch
    launches_per_step = ctx.kernel_launches() - l0
    out_ranks = out.ranks()
    del out
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    o = eager_step()
    e1.record(stream)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    del o

    # CUDA-graph plan of the same call (what the timed loop replays)
    plan = P.FixedKrpPlan(y, ranks, seed)

    def step():
        plan.execute()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (inputs 18 GB >> 126 MB L2: no flush needed) ----
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly the timed steps
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    launches = ctx.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = flops * world / (ms * 1e-3) / 1e12

    # ---- phase timing (separate step; events around each phase) ----
    C_ = P.lib()
    C_.ttr_ctx_enable_timing(ctx._h, 1)
    C_.ttr_ctx_phase_times(ctx._h, None, None)
    o = eager_step()
    del o
    phase_ms = (C.c_double * 4)()
    phase_n = (C.c_uint64 * 4)()
    C_.ttr_ctx_phase_times(ctx._h, phase_ms, phase_n)
    C_.ttr_ctx_enable_timing(ctx._h, 0)
    sketch_ms = phase_ms[0]
    achieved = sketch_flops / (sketch_ms * 1e-3) / 1e12 if sketch_ms > 0 else None

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        n_, r_, total = y.shape()
        host_in = torch.empty(total, dtype=torch.float64, pin_memory=True)
        C_.ttr_tt_download(ctx._h, y._h, C.c_void_p(host_in.data_ptr()))
        _, _, out_total = plan.output.shape()
        host_out = torch.empty(out_total, dtype=torch.float64, pin_memory=True)
        reps = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        # (a) serial: H2D, graph replay, D2H one after the other
        times = []
        for it in range(reps + 1):
            t0 = time.perf_counter()
            C_.ttr_tt_copy_from_host(ctx._h, y._h, C.c_void_p(host_in.data_ptr()))  # H2D from pinned memory
            plan.execute()
            C_.ttr_tt_download(ctx._h, plan.output._h, C.c_void_p(host_out.data_ptr()))  # D2H + sync
            dt = time.perf_counter() - t0
            if it > 0:
                times.append(dt)
        serial_ms = sum(times) / len(times) * 1e3
        ref_out = host_out.clone()
        # (b) host-streaming plan (ttr_plan_fixed_krp_host): the copies are graph
        # nodes on a copy stream overlapped with the sketch / sweep
        hplan = P.FixedKrpPlan(y, ranks, 7, host_in=host_in, host_out=host_out)
        times = []
        for it in range(reps + 1):
            host_out.zero_()
            t0 = time.perf_counter()
            hplan.execute()
            ctx.synchronize()
            dt = time.perf_counter() - t0
            if it > 0:
                times.append(dt)
        e2e_ms = sum(times) / len(times) * 1e3
        e2e_bitwise = bool(torch.equal(ref_out, host_out))
        hplan.close()
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": flops * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": 8 * out_total,
               "timing": "host wall clock around ttr_plan_execute of a host-streaming plan "
                         "(ttr_plan_fixed_krp_host: pinned H2D of the cores and D2H of the result as graph nodes "
                         "overlapped with the sweep) + ttr_ctx_synchronize",
               "serial_ms_per_step": serial_ms, "bitwise_equal_to_serial": e2e_bitwise}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_full_fixed(P, y, ranks, seed, cfg, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device Philox Gaussian cores)",
            "config": {"workload": f"config {args.config} fixed-rank KRP rounding round_fixed_krp(Y, {{{cfg['ell']}}}x{cfg['d'] - 1}, 7)",
                       "d": cfg["d"], "n": cfg["n"], "formal_rank": cfg["rx"] + cfg["rz"], "l": cfg["ell"],
                       "input_gb": total_bytes(y) / 1e9, "output_ranks": out_ranks,
                       "flops_per_step": flops, "sketch_flops_per_step": sketch_flops,
                       "api": "FixedKrpPlan (CUDA graph of round_fixed_krp) replayed per step",
                       "eager_ms_per_step": eager_ms,
                       "l2": {"5b": "inputs exceed L2 (18 GB vs 126 MB)", "3": "inputs exceed L2 (2.3 GB)",
                              "1": "3.2 MB input is L2-resident (a step re-reads cores from L2; config 1 is "
                                   "launch/latency bound)"}[args.config],
                       "parallelism": f"{world} independent tensors (batch sharding)"},
            "tflops_fp64": value, "fraction_of_fp64_peak": value / world / FP64_PEAK_TFLOPS,
            "phase_ms": {"sketch": phase_ms[0], "qr": phase_ms[1], "lr_gemm": phase_ms[2], "other": phase_ms[3]},
            "roofline": roofline_entry(achieved, cfg, sketch_ms / (cfg["d"] - 1) if sketch_ms > 0 else None),
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "gpu_launches_per_step": launches_per_step,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# `ncu --set full` of one sketch launch at the 5b middle-core shape (tools/sketch_profile.py +
# tools/ncu_to_json.py): this round's capture, else round 1's (the kernel is unchanged)
SKETCH_NCU = [os.path.join(ROOT, "profiles", f) for f in ("r02f_ncu_sketch_tma.json", "r01_ncu_sketch_tma.json")]


HBM_PEAK_GBS = 6534.5  # MEASURED_PEAKS.json (copy bandwidth of this pool's B200)
RIDGE = FP64_PEAK_TFLOPS * 1e12 / (HBM_PEAK_GBS * 1e9)  # flop/B


def roofline_entry(achieved, cfg, ms_per_launch=None):
    """Sketch-kernel roofline: achieved = algorithmic flops of the d-1 krp_step launches
    / their CUDA-event time; traffic = DRAM bytes (read + write) of ONE middle-core
    launch from the committed `ncu --set full` capture at the same shape. The sketch's
    arithmetic intensity is l/4 flop/B: below the ridge (config 1, l = 15) the bound is
    HBM and `achieved` is the algorithmic bytes (every core read once) per launch time."""
    r = cfg["rx"] + cfg["rz"]
    abytes = 8 * (r * cfg["n"] * r + r * cfg["ell"] + cfg["n"] * cfg["ell"] + r * cfg["ell"])
    if cfg["ell"] / 4 < RIDGE and ms_per_launch:
        gbs = abytes / (ms_per_launch * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": gbs, "peak": HBM_PEAK_GBS, "unit": "GB/s", "frac": gbs / HBM_PEAK_GBS,
                "traffic": None, "kernel": "krp_step (KRP sketch contraction, cp.async DMMA kernel)",
                "peak_source": "MEASURED_PEAKS.json HBM copy bandwidth",
                "algorithmic_bytes_per_launch": abytes,
                "note": "average over the d-1 sketch launches (phase time incl. their split-K reduce / transpose "
                        "launches); at config 1's size (0.4 MB per core) every launch is latency-bound"}
    entry = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
             "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": None,
             "kernel": "krp_step: dgemm_tma_kernel<128,64,KM=1> (TMA + mbarrier pipeline, fp64 DMMA) + "
                       "splitk_reduce_wide",
             "peak_source": PEAK_SOURCE,
             "algorithmic_bytes_per_launch": abytes}
    if (cfg["n"], r, cfg["ell"]) != (128, 1000, 320):
        return entry  # the committed capture is at the 5b shape only
    for path in SKETCH_NCU:
        try:
            with open(path) as f:
                ncu = json.load(f)
            entry["traffic"] = ncu["dram_read_bytes"] + ncu["dram_write_bytes"]
            entry["traffic_unit"] = "bytes per launch (middle core)"
            entry["traffic_source"] = f"profiles/{os.path.basename(path)} (ncu --set full, same shape; the write " \
                                      "share is the deterministic split-K partials)"
            entry["ncu_dmma_pipe_active_pct"] = ncu.get("dmma_pipe_active_pct")
            break
        except (OSError, KeyError, ValueError):
            continue
    return entry


def total_bytes(y):
    return 8 * y.shape()[2]


def cpu_full_fixed(P, y, ranks, seed, cfg, args):
    """cpu_baseline: the CPU oracle (reference restatement, OpenBLAS backend, all host
    threads) on the FULL config input (downloaded from the device), one round."""
    O = _oracle()
    threads = cpu_threads(args)
    with O.backend_scope("blas", threads):
        n, r, _ = y.shape()
        x = O.TT.from_flat(len(n), n, r, y.flat())
        sec, fl = cpu_round(O, x, ranks, seed)
    return {"value": fl / sec / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
            "sample": cpu_desc(cfg, threads), "seconds": sec, "ms_per_round": sec * 1e3, "same_config": True}


ADAPTIVE = {
    "2": dict(d=16, n=32, rx=30, rz=170, eps=1e-6, seed=1002, tol=1e-4, f_init=0.1, f_inc=0.05,
              desc="config 2 adaptive KRP rounding round_adaptive_krp(Y, {tol 1e-4, f_init 0.1, f_inc 0.05, seed 7}); "
                   "Y = X/|X| + 1e-6 Z/|Z|, d=16, n=32, ranks 30 + 170"),
    "4": dict(d=12, n=128, terms=20, r=20, ell_k=0.3, seed=1004, tol=1e-6, f_init=0.1, f_inc=0.04,
              desc="config 4 adaptive KRP rounding round_adaptive_krp(Y, {tol 1e-6, f_init 0.1, f_inc 0.04, seed 7}); "
                   "Y = sum of 20 rank-20 exp(-|t-c|/0.3) TTs weighted 2^-i, d=12, n=128"),
}


def run_adaptive(args, world, rank, local):
    """Configs 2 and 4: adaptive-rank KRP rounding. One step = one round_adaptive_krp through its
    CUDA-graph plan (the eager call's time is reported beside it); independent tensor per rank
    (weak scaling)."""
    import torch
    import paper_2511_03598_b200 as P
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local, stream.cuda_stream)
    a = ADAPTIVE[args.config]
    if args.config == "2":
        y = P.TTTensor.two_part_philox(a["d"], a["n"], a["rx"], a["rz"], a["eps"], a["seed"] + 1000 * rank, ctx)
    else:
        y = P.TTTensor.kernel_sum(a["d"], a["n"], a["r"], a["terms"], a["ell_k"], a["seed"] + 1000 * rank, ctx)
    cfgA = P.AdaptiveConfig(tolerance=a["tol"], f_init=a["f_init"], f_inc=a["f_inc"], seed=7)
    ctx.reset_counters()
    l0 = ctx.kernel_launches()
    out = P.round_adaptive_krp(y, cfgA)
    torch.cuda.synchronize()
    flops = ctx.counters().total()
    launches_per_step = ctx.kernel_launches() - l0
    out_ranks = out.ranks()
    del out
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # the eager call (host-side growth decisions), timed for reference
    for _ in range(args.warmup):
        del_ = P.round_adaptive_krp(y, cfgA)
        del del_
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        o = P.round_adaptive_krp(y, cfgA)
        del o
    e1.record(stream)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / args.steps
    # the timed API: the CUDA-graph plan (ttr_plan_adaptive_krp) — the recorded growth
    # decisions replayed by one graph launch and re-checked on the device per step
    plan = P.AdaptiveKrpPlan(y, cfgA)
    for _ in range(args.warmup):
        plan.execute()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            plan.execute()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / args.steps
    plan_equal = bool(np.array_equal(plan.output.flat(), P.round_adaptive_krp(y, cfgA).flat()))
    rerecords = plan.rerecords()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # roofline: the initial KRP sketch contraction (estimate_norm_krp at the initial width:
    # all d-1 contractions + V(X_1) W_2), CUDA events on the context stream
    n, r, total = y.shape()
    w = math.ceil(a["f_init"] * max(r))
    ctx.reset_counters()
    P.estimate_norm_krp(y, w, 7)
    sk_flops = ctx.counters().total()
    reps = 5
    e0.record(stream)
    for _ in range(reps):
        P.estimate_norm_krp(y, w, 7)
    e1.record(stream)
    torch.cuda.synchronize()
    sk_ms = e0.elapsed_time(e1) / reps
    sk_bytes = 8 * total  # every core read once
    ai = sk_flops / sk_bytes
    if ai < RIDGE:
        gbs = sk_bytes / (sk_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": HBM_PEAK_GBS, "unit": "GB/s", "frac": gbs / HBM_PEAK_GBS,
                "peak_source": "MEASURED_PEAKS.json HBM copy bandwidth"}
    else:
        tf = sk_flops / (sk_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tf / FP64_PEAK_TFLOPS, "peak_source": PEAK_SOURCE}
    roof.update({"traffic": None, "kernel": f"initial KRP sketch (estimate_norm_krp, width {w}): d-1 krp_step launches",
                 "algorithmic_bytes_per_launch": sk_bytes, "algorithmic_flops": sk_flops, "ms": sk_ms,
                 "arithmetic_intensity": ai})

    # e2e through the API with host buffers: pinned H2D of the cores, the rounding, D2H of the result
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty(total, dtype=torch.float64, pin_memory=True)
        P.lib().ttr_tt_download(ctx._h, y._h, C.c_void_p(host_in.data_ptr()))
        times, out_bytes = [], 0
        for it in range(min(args.steps, 3) + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.lib().ttr_tt_copy_from_host(ctx._h, y._h, C.c_void_p(host_in.data_ptr()))
            plan.execute()
            o = plan.output
            _, _, ot = o.shape()
            host_out = torch.empty(ot, dtype=torch.float64, pin_memory=True) if it == 0 else host_out
            P.lib().ttr_tt_download(ctx._h, o._h, C.c_void_p(host_out.data_ptr()))
            dt = time.perf_counter() - t0
            out_bytes = 8 * ot
            del o
            if it > 0:
                times.append(dt)
        e2e_ms = sum(times) / len(times) * 1e3
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": flops * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": out_bytes,
               "timing": "host wall clock: pinned H2D of the cores (ttr_tt_copy_from_host) + the adaptive plan's "
                         "execute (graph replay + device-side decision check) + D2H of the result (ttr_tt_download)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        O = _oracle()
        x = O.TT.from_flat(len(n), n, r, y.flat())
        O.flops_reset()
        t0 = time.perf_counter()
        ref = O.round_adaptive_krp(x, tolerance=a["tol"], f_init=a["f_init"], f_inc=a["f_inc"], seed=7, rng=O.PHILOX)
        sec = time.perf_counter() - t0
        cfl = sum(v for k, v in O.flops_get().items() if k in ("gemm", "qr", "svd"))
        cpu = {"value": cfl / sec / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
               "sample": "the full config: round_adaptive_krp on the same input, CPU oracle, wall clock around the call",
               "seconds": sec, "ms_per_round": sec * 1e3, "ranks_identical": ref.ranks == out_ranks}

    if rank == 0:
        line = {
            "metric": METRIC, "value": flops * world / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated input)",
            "config": {"workload": a["desc"], "output_ranks": out_ranks, "flops_per_step": flops,
                       "input_gb": 8 * total / 1e9,
                       "api": "AdaptiveKrpPlan (ttr_plan_adaptive_krp: CUDA graph of round_adaptive_krp with the "
                              "recorded growth decisions, each re-checked on the device) replayed per step",
                       "eager_ms_per_step": eager_ms, "plan_bitwise_equal_eager": plan_equal,
                       "plan_rerecords": rerecords,
                       "l2": "inputs exceed L2" if 8 * total > 126e6 else "input fits L2 (126 MB); not flushed",
                       "parallelism": f"{world} independent tensors"},
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": launches,
            "gpu_launches_per_step": launches_per_step, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args, world, rank, local):
    """Config 5b, ONE tensor over N GPUs (csrc/sharded.cu through
    ttr_round_fixed_krp_sharded): column-sharded KRP sketch + NCCL all-gather of the
    W slices, row-sharded Rand-Orth sweep with a TSQR per mode. Every rank holds a
    replica of the input; the output stays sharded (rank p: the core slices J_p).
    value = the job's algorithmic flops (one round_fixed_krp, the reference's
    charges) / max-over-ranks time. Strong scaling."""
    import torch
    import paper_2511_03598_b200 as P
    from paper_2511_03598_b200.distributed import Communicator, round_fixed_krp_sharded
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local, stream.cuda_stream)
    cfg = dict(CFG5B)
    y = build_input(P, ctx, cfg)  # identical replica on every rank
    ranks = [cfg["ell"]] * (cfg["d"] - 1)
    seed = cfg["round_seed"]
    # the job's work = one round_fixed_krp with the reference's charges
    ctx.reset_counters()
    o = P.round_fixed_krp(y, ranks, seed)
    torch.cuda.synchronize()
    flops_job = ctx.counters().total()
    out_ranks = o.ranks()
    del o
    if args.local_ranks:
        comm = Communicator.local(ctx, args.local_ranks)
    elif world > 1:
        comm = Communicator.from_torch(ctx)
    else:
        comm = Communicator.local(ctx, 1)

    def step():
        loc, _ = round_fixed_krp_sharded(y, ranks, seed, comm, gather=False)
        return loc

    ctx.reset_counters()
    l0 = ctx.kernel_launches()
    step()
    launches_per_step = ctx.kernel_launches() - l0
    flops_rank = ctx.counters().total()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = flops_job / (ms * 1e-3) / 1e12

    e2e = None
    if not args.no_e2e:
        # through the API with host buffers: H2D of this rank's input replica from pinned
        # memory, the sharded round, D2H of this rank's output shard
        n_, r_, total = y.shape()
        host_in = torch.empty(total, dtype=torch.float64, pin_memory=True)
        P._check(P.lib().ttr_tt_download(ctx._h, y._h, C.c_void_p(host_in.data_ptr())))
        reps = max(1, min(args.steps, 3))
        times, d2h = [], 0
        for it in range(reps + 1):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            P._check(P.lib().ttr_tt_copy_from_host(ctx._h, y._h, C.c_void_p(host_in.data_ptr())))
            loc = step()
            d2h = 0
            for lt in loc:
                if lt is not None:
                    f = lt.flat()
                    d2h += 8 * f.size
            dt = time.perf_counter() - t0
            if it > 0:
                times.append(dt)
        e2e_ms = sum(times) / len(times) * 1e3
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": flops_job / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": d2h,
               "timing": "host wall clock per rank (max over ranks): pinned H2D of the input replica "
                         "(ttr_tt_copy_from_host), ttr_round_fixed_krp_sharded, D2H of the rank's output shard"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device Philox Gaussian cores)",
            "config": {"workload": "config 5b, ONE tensor over the GPUs: column-sharded KRP sketch + NCCL "
                                   "all-gather, row-sharded Rand-Orth sweep with an NVLink TSQR per mode "
                                   "(ttr_round_fixed_krp_sharded)",
                       "d": cfg["d"], "n": cfg["n"], "formal_rank": cfg["rx"] + cfg["rz"], "l": cfg["ell"],
                       "output_ranks": out_ranks, "flops_per_step": flops_job, "flops_per_rank": flops_rank,
                       "local_ranks": args.local_ranks or None, "l2": "inputs exceed L2 (18 GB vs 126 MB)",
                       "parallelism": f"{world} GPUs, one tensor (columns of the sketch, rows of the sweep)"},
            "tflops_fp64": value, "fraction_of_fp64_peak": value / world / FP64_PEAK_TFLOPS,
            "clocks": clk.summary(), "gpu_launches": launches, "gpu_launches_per_step": launches_per_step,
            "e2e": e2e, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_5a(args, world, rank, local):
    """Config 5a: 4096 independent tensors (d=8, n=16, rank 16 + 1e-6 rank 48 -> 64, l=20), the
    batch split across ranks (strong scaling, no collective); one step rounds the whole batch."""
    import torch
    import paper_2511_03598_b200 as P
    from paper_2511_03598_b200.seeds import derive_seed
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local, stream.cuda_stream)
    total_batch = 4096
    nb = total_batch // world + (1 if rank < total_batch % world else 0)
    batch = P.TTBatch.two_part_philox(nb, 8, 16, 16, 48, 1e-6, derive_seed(1005, 1000 + rank), ctx)
    ranks = [20] * 7
    ctx.reset_counters()
    o = P.round_fixed_krp_batched(batch, ranks, 7)
    torch.cuda.synchronize()
    flops = ctx.counters().total()
    out_ranks = o.shape()[2]
    del o
    for _ in range(args.warmup):
        o = P.round_fixed_krp_batched(batch, ranks, 7)
        del o
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        torch.cuda.profiler.start()  # scopes `ncu --profile-from-start off` to the timed steps
        e0.record(stream)
        for _ in range(args.steps):
            o = P.round_fixed_krp_batched(batch, ranks, 7)
            del o
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    launches = ctx.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    flops_all = flops * world  # per-rank work is (near) equal

    # roofline: the fused next-core + next-sketch kernel (lr_fused_kernel, the "other"
    # phase of the batched sweep; d-2 launches per step), CUDA events on the stream
    _, n_, r_in, _ = batch.shape()
    rb = out_ranks
    C_ = P.lib()
    C_.ttr_ctx_enable_timing(ctx._h, 1)
    C_.ttr_ctx_phase_times(ctx._h, None, None)
    o = P.round_fixed_krp_batched(batch, ranks, 7)
    del o
    phase_ms = (C.c_double * 4)()
    phase_n = (C.c_uint64 * 4)()
    C_.ttr_ctx_phase_times(ctx._h, phase_ms, phase_n)
    C_.ttr_ctx_enable_timing(ctx._h, 0)
    d_ = len(n_)
    fb, ff = 0, 0  # algorithmic bytes / flops of the d-2 fused launches
    for k in range(1, d_ - 1):
        l, cols, nk, rr, l2 = rb[k], r_in[k], n_[k], r_in[k + 1], rb[k + 1]
        # X read, Y write, S (or, fused with the next QR, Q) write, M read, W read,
        # and the fused kernel's M_next write (l2 x rr)
        fb += 8 * nb * (cols * nk * rr + l * nk * rr + l * nk * l2 + l * cols + rr * l2 + l2 * rr)
        ff += nb * (2 * l * nk * rr * cols + 2 * l * nk * l2 * rr)
    fused_ms = phase_ms[3]
    roof = None
    if fused_ms > 0:
        gbs = fb / (fused_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": HBM_PEAK_GBS, "unit": "GB/s", "frac": gbs / HBM_PEAK_GBS,
                "traffic": None, "kernel": "lr_fused_kernel<3,3,10> (next core M H(X) + next sketch V(Y) W + its Householder "
                                          "QR (the output core) + M_next = Q^T V(Y), one CTA per tensor, "
                                          "cp.async-streamed X slices, fp64 DMMA)",
                "peak_source": "MEASURED_PEAKS.json HBM copy bandwidth",
                "algorithmic_bytes_per_launch": fb / (d_ - 2), "launches": d_ - 2, "ms_all_launches": fused_ms,
                "arithmetic_intensity": ff / fb, "tflops_achieved": ff / (fused_ms * 1e-3) / 1e12}
        try:
            with open(os.path.join(ROOT, "profiles", "r01_ncu_lr_fused.json")) as f:
                nc = json.load(f)
            roof["traffic"] = nc["dram_read_bytes"] + nc["dram_write_bytes"]
            roof["traffic_source"] = "profiles/r01_ncu_lr_fused.json (ncu --set full of one middle-mode launch)"
            roof["ncu_dmma_pipe_active_pct"] = nc.get("dmma_pipe_active_pct")
        except (OSError, KeyError, ValueError):
            pass

    # e2e through the C ABI with host buffers: pinned H2D of the whole batch (ttr_batch_upload),
    # the batched rounding, D2H of every rounded tensor (ttr_batch_download)
    e2e = None
    if not args.no_e2e:
        tot_in = batch.shape()[3]
        host_in = torch.empty(nb * tot_in, dtype=torch.float64, pin_memory=True)
        C_.ttr_batch_download(ctx._h, batch._h, C.c_int64(0), C.c_int64(nb), C.c_void_p(host_in.data_ptr()))
        host_out = None
        times = []
        for it in range(min(args.steps, 3) + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hb = C.c_void_p()
            P._check(C_.ttr_batch_upload(ctx._h, C.c_int64(nb), C.c_int64(d_), P._i64(n_), P._i64(r_in),
                                         C.c_void_p(host_in.data_ptr()), C.byref(hb)))
            up = P.TTBatch(hb, ctx)
            o = P.round_fixed_krp_batched(up, ranks, 7)
            tot_out = o.shape()[3]
            if host_out is None:
                host_out = torch.empty(nb * tot_out, dtype=torch.float64, pin_memory=True)
            C_.ttr_batch_download(ctx._h, o._h, C.c_int64(0), C.c_int64(nb), C.c_void_p(host_out.data_ptr()))
            dt = time.perf_counter() - t0
            del o, up
            if it > 0:
                times.append(dt)
        e2e_ms = sum(times) / len(times) * 1e3
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": flops_all / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * nb * tot_in, "d2h_bytes_per_step": 8 * nb * tot_out,
               "timing": "host wall clock: ttr_batch_upload (pinned H2D of all tensors) + "
                         "ttr_round_fixed_krp_batched + ttr_batch_download (synchronising)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        O = _oracle()
        sample = 128
        xs = [O.TT.from_flat(d_, n_, r_in, f) for f in batch.flats(0, sample)]
        O.flops_reset()
        t0 = time.perf_counter()
        for b, x in enumerate(xs):
            O.round_fixed_krp(x, ranks, O.derive_seed(7, b), rng=O.PHILOX)
        sec = time.perf_counter() - t0
        fl = O.flops_get()["total"]
        cpu = {"value": fl / sec / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"round_fixed_krp of the first {sample} tensors of the batch (same inputs and per-tensor "
                         f"seeds), CPU oracle, wall clock around the loop", "seconds": sec,
               "ms_per_4096_tensors_extrapolated": sec / sample * 4096 * 1e3}

    if rank == 0:
        line = {
            "metric": METRIC, "value": flops_all / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (device Philox Gaussian cores)",
            "config": {"workload": "config 5a: 4096 x round_fixed_krp(Y_b, {20}x7, derive_seed(7,b)), batched",
                       "batch_per_rank": nb, "output_ranks": out_ranks, "flops_per_step_per_rank": flops,
                       "bytes_per_step": 8 * 4096 * batch.shape()[3],
                       "l2": "inputs exceed L2 (12.9 GB)"},
            "hbm_gbs_achieved": 8 * 4096 * batch.shape()[3] / (ms * 1e-3) / 1e9,
            "phase_ms": {"sketch": phase_ms[0], "qr": phase_ms[1], "gemm": phase_ms[2], "fused_sweep": phase_ms[3]},
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    maybe_spawn(args)
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.config == "5a":
        run_5a(args, world, rank, local)
        return
    if args.config in ADAPTIVE:
        run_adaptive(args, world, rank, local)
        return
    if args.config == "5b" and (args.local_ranks or (world > 1 and args.sharding == "tensor")):
        run_sharded(args, world, rank, local)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
