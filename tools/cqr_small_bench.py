"""Micro-benchmark of the batched small sCQR3 (qr_chol.cu K4e) through the C ABI:
time per call of `batch` m x n matrices, orthogonality and residual.
Usage: python tools/cqr_small_bench.py [batch]"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402

L = P.lib()
L.ttr_dev_thin_qr_cholesky_batched.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                               C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]


def run(ctx, batch, m, n, reps=20, decades=6):
    a = torch.randn(batch, n, m, dtype=torch.float64, device="cuda")  # column-major m x n each
    a[:, :, :] *= torch.logspace(0, -decades, n, dtype=torch.float64, device="cuda")[None, :, None]
    q = torch.empty_like(a)
    f = torch.zeros(batch, dtype=torch.int32, device="cuda")
    call = lambda: L.ttr_dev_thin_qr_cholesky_batched(ctx._h, m, n, batch, a.data_ptr(), m, m * n, q.data_ptr(), m,
                                                      m * n, f.data_ptr())
    for _ in range(3):
        assert call() == 0, L.ttr_last_error()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    qm = q.transpose(1, 2)  # batch x m x n
    am = a.transpose(1, 2)
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    orth = torch.linalg.norm(qm.transpose(1, 2) @ qm - eye, dim=(1, 2)).max().item()
    res = (torch.linalg.norm(qm @ (qm.transpose(1, 2) @ am) - am, dim=(1, 2)) / torch.linalg.norm(am, dim=(1, 2))).max().item()
    print(f"cqr_small batch {batch} {m}x{n} kappa 1e{decades}: {ms * 1e3:.1f} us/call  {ms * 1e3 / batch * 148:.2f} us per tensor-slot  "
          f"orth {orth:.2e} resid {res:.2e} broken {int(f.sum().item())}", flush=True)


if __name__ == "__main__":
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    ctx = P.default_context()
    for m, n in [(320, 20), (256, 20), (320, 16), (512, 32), (64, 8), (101, 13)]:
        run(ctx, batch, m, n)
    run(ctx, batch, 320, 20, decades=11)
