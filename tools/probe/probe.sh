#!/bin/bash
# Box probe: host cores, GPU identity, fp64 peaks (DFMA, DMMA, cuBLAS DGEMM).
# Run under gpurun; writes gpurun_out/probe.log.
set -x
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
{
  nproc; lscpu | head -30; free -g; numactl -H 2>/dev/null | head -5
  nvidia-smi
  nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv
  ./tools/probe/fp64_peak
  python - <<'EOF'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(3): c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print('{"probe": "cublas_dgemm_8192", "ms": %.3f, "tflops": %.3f}' % (best, 2 * 8192**3 / (best * 1e-3) / 1e12))
for m, n, k in [(40960, 320, 1000), (320, 128000, 1000), (1000, 320, 128000), (25600, 400, 400)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print('{"probe": "cublas_dgemm_%dx%dx%d", "ms": %.3f, "tflops": %.3f}' % (m, n, k, best, 2 * m * n * k / (best * 1e-3) / 1e12))
# QR probe (cuSOLVER through torch) for tall-skinny
for m, n in [(40960, 320), (7040, 110)]:
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for _ in range(2): q, r = torch.linalg.qr(a)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); q, r = torch.linalg.qr(a); e1.record(); torch.cuda.synchronize()
    print('{"probe": "torch_qr_%dx%d", "ms": %.3f}' % (m, n, e0.elapsed_time(e1)))
EOF
} > gpurun_out/probe.log 2>&1
echo done
