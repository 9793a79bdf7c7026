"""Run the device thin QR once per shape (after a warm-up call) — for ncu launch lists:
ncu --metrics gpu__time_duration.sum --csv python tools/qr_once.py m n [m n ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    L = P.lib()
    shapes = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(1, len(sys.argv) - 1, 2)]
    for m, n in shapes:
        a = torch.randn(n, m, dtype=torch.float64, device="cuda")
        q = torch.empty(n, m, dtype=torch.float64, device="cuda")
        for _ in range(2):
            P._check(L.ttr_dev_thin_qr(ctx._h, P.C.c_int64(m), P.C.c_int64(n), P.C.c_void_p(a.data_ptr()),
                                       P.C.c_int64(m), P.C.c_void_p(q.data_ptr()), P.C.c_int64(m), None,
                                       P.C.c_int64(1)))
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
