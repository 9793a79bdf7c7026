"""Diagnostics for the deterministic TT-SVD path (config 3): per-call SVD sweep
counts (TTR_SVD_TRACE) and the phase split. Usage: TTR_SVD_TRACE=1 python tools/det_trace.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream.cuda_stream)
y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    z = P.round_deterministic(y, target_ranks=[100] * 29)
    torch.cuda.synchronize()
    print("det ms", (time.perf_counter() - t) * 1e3, flush=True)
