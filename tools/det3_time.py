"""Config 3's comparison call round_deterministic(Y, {100}x29) timed on the GPU
(CUDA events, after a warm-up call) and, with --cpu, on the host oracle
(OpenBLAS backend, all threads). Prints one JSON line."""
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2511_03598_b200 as P  # noqa: E402


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
    ranks = [100] * 29
    P.round_deterministic(y, target_ranks=ranks)
    ctx.reset_counters()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = P.round_deterministic(y, target_ranks=ranks)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fl = ctx.counters().total()
    rec = {"workload": "config 3 round_deterministic(Y, {100}x29)", "gpu_ms": ms, "flops": fl,
           "gpu_tflops": fl / (ms * 1e-3) / 1e12, "ranks": out.ranks()}
    if "--cpu" in sys.argv:
        import py_oracle as O
        threads = os.cpu_count() or 1
        with O.backend_scope("blas", threads):
            n, r, _ = y.shape()
            x = O.TT.from_flat(len(n), n, r, y.flat())
            t0 = time.perf_counter()
            O.round_deterministic(x, ranks=ranks)
            rec["cpu_s"] = time.perf_counter() - t0
            rec["cpu_threads"] = threads
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
