"""Adaptive rounding (config 4, or config 2 with argument "2") under
ncu --profile-from-start off (third call only)."""
import sys, os, torch, time
sys.path.insert(0, '/root/repo')
import paper_2511_03598_b200 as P
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = P.Context(0, stream.cuda_stream)
if len(sys.argv) > 1 and sys.argv[1] == "2":
    y = P.TTTensor.two_part_philox(16, 32, 30, 170, 1e-6, 1002, ctx)
    c = P.AdaptiveConfig(tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7)
else:
    y = P.TTTensor.kernel_sum(12, 128, 20, 20, 0.3, 1004, ctx)
    c = P.AdaptiveConfig(tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    if i == 2: torch.cuda.profiler.start()
    o = P.round_adaptive_krp(y, c)
    torch.cuda.synchronize()
    if i == 2: torch.cuda.profiler.stop()
    print("ms", (time.perf_counter() - t) * 1e3, "launches", ctx.kernel_launches())
