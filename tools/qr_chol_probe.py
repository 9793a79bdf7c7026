"""Launch-list probe of the shifted Cholesky QR (run under ncu): two calls per shape."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402

L = P.lib()
L.ttr_dev_thin_qr_cholesky.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
bd = C.c_int(0)
shapes = [(40960, 320), (7040, 110), (6400, 400)]
if len(sys.argv) > 2:
    shapes = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(1, len(sys.argv) - 1, 2)]
for m, n in shapes:
    a = torch.randn(n, m, dtype=torch.float64, device="cuda")
    q = torch.empty_like(a)
    for _ in range(2):
        L.ttr_dev_thin_qr_cholesky(ctx._h, m, n, a.data_ptr(), m, q.data_ptr(), m, None, 1, C.byref(bd))
