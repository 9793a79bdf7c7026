"""Secondary measurements: every BASELINE config on one B200 through the C ABI
(eager API; fixed-rank configs also through the CUDA-graph plan).
Prints one JSON line per config: ms per call (CUDA events on the context
stream, median of reps after warm-up), algorithmic TFLOP/s (reference charges),
output ranks."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402


def timed(ctx, stream, fn, reps, warm=2):
    for _ in range(warm):
        out = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.reset_counters()
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), ctx.counters().total(), out


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    which = sys.argv[1:] or ["1", "2", "3", "3rot", "3det", "4", "4sum"]
    for cfg in which:
        if cfg == "1":
            y = P.TTTensor.two_part_philox(10, 20, 10, 40, 1e-4, 1001, ctx)
            plan = P.FixedKrpPlan(y, [15] * 9, 7)
            ms, fl, _ = timed(ctx, stream, lambda: P.round_fixed_krp(y, [15] * 9, 7), 5)
            msp, _, _ = timed(ctx, stream, lambda: plan.execute(), 20)
            rec = dict(config="1 fixed KRP d=10 n=20 50->15", ms_eager=ms, ms_plan=msp, tflops=fl / msp / 1e9,
                       ranks=plan.output.ranks())
        elif cfg == "2":
            y = P.TTTensor.two_part_philox(16, 32, 30, 170, 1e-6, 1002, ctx)
            c = P.AdaptiveConfig(tolerance=1e-4, f_init=0.1, f_inc=0.05, seed=7)
            ms, fl, out = timed(ctx, stream, lambda: P.round_adaptive_krp(y, c), 3)
            rec = dict(config="2 adaptive KRP d=16 n=32 200, tol 1e-4", ms_eager=ms, tflops=fl / ms / 1e9,
                       ranks=out.ranks())
        elif cfg == "3":
            y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
            plan = P.FixedKrpPlan(y, [110] * 29, 7)
            msp, fl, _ = timed(ctx, stream, lambda: plan.execute(), 5)
            rec = dict(config="3 fixed KRP d=30 n=64 400->110", ms_plan=msp, tflops=fl / msp / 1e9,
                       ranks=plan.output.ranks()[:4])
        elif cfg == "3rot":
            # the paper's baseline: Rand-Orth with a Gaussian TT sketch, same input and ranks
            y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
            ms, fl, out = timed(ctx, stream, lambda: P.round_rand_orth_tt(y, [110] * 29, 7), 3)
            ctx.reset_counters()
            P.round_rand_orth_tt(y, [110] * 29, 7)
            sk = ctx.counters().sketch
            rec = dict(config="3 Rand-Orth TT sketch d=30 n=64 400->110", ms_eager=ms, tflops=fl / ms / 1e9,
                       sketch_flops=sk, ranks=out.ranks()[:4])
        elif cfg == "3det":
            y = P.TTTensor.two_part_philox(30, 64, 100, 300, 1e-8, 1003, ctx)
            ms, fl, out = timed(ctx, stream, lambda: P.round_deterministic(y, target_ranks=[100] * 29), 1, warm=1)
            rec = dict(config="3 deterministic TT-SVD d=30 n=64 400->100", ms_eager=ms, tflops=fl / ms / 1e9,
                       ranks=out.ranks()[:4])
        elif cfg == "4":
            y = P.TTTensor.kernel_sum(12, 128, 20, 20, 0.3, 1004, ctx)
            c = P.AdaptiveConfig(tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7)
            ms, fl, out = timed(ctx, stream, lambda: P.round_adaptive_krp(y, c), 3)
            rec = dict(config="4 adaptive KRP d=12 n=128 kernel-sum 400, tol 1e-6", ms_eager=ms,
                       tflops=fl / ms / 1e9, ranks=out.ranks())
        elif cfg == "3sum":
            # config-3 input kept as its two summands: round_sum_adaptive_krp (no formal
            # sum, one sketch per term) vs round_adaptive_krp of the formal sum, tol 1e-6
            from paper_2511_03598_b200.seeds import derive_seed
            modes = [64] * 30
            x = P.TTTensor.random_philox(modes, [1] + [100] * 29 + [1], derive_seed(1003, 1), ctx)
            z = P.TTTensor.random_philox(modes, [1] + [300] * 29 + [1], derive_seed(1003, 2), ctx)
            x = P.scaled(x, 1.0 / P.norm_exact(x))
            z = P.scaled(z, 1e-8 / P.norm_exact(z))
            y = P.formal_sum([x, z])
            ms_s, fl_s, out_s = timed(ctx, stream, lambda: P.round_sum_adaptive_krp([x, z], 1e-6, 0.05, 7), 3)
            c = P.AdaptiveConfig(tolerance=1e-6, f_init=0.25, f_inc=0.05, seed=7)
            ms_f, fl_f, out_f = timed(ctx, stream, lambda: P.round_adaptive_krp(y, c), 3)
            rec = dict(config="3sum adaptive tol 1e-6, d=30 n=64, X(100) + 1e-8 Z(300)", ms_sum=ms_s,
                       tflops_sum=fl_s / ms_s / 1e9, ranks_sum=out_s.ranks()[:4], ms_formal=ms_f,
                       tflops_formal=fl_f / ms_f / 1e9, ranks_formal=out_f.ranks()[:4],
                       sketch_flop_ratio=(100 ** 2 + 300 ** 2) / 400 ** 2,
                       rel_diff=P.relative_error(out_f, out_s))
        elif cfg == "4sum":
            # config 4's input IS a sum of 20 rank-20 terms: round it without the formal
            # sum (one 20-rank sketch per term) vs the formal-sum adaptive rounding
            terms = [P.TTTensor.kernel_term(12, 128, 20, t, 0.3, 1004, ctx) for t in range(20)]
            y = P.formal_sum(terms)
            ms_s, fl_s, out_s = timed(ctx, stream, lambda: P.round_sum_adaptive_krp(terms, 1e-6, 0.04, 7), 3)
            c = P.AdaptiveConfig(tolerance=1e-6, f_init=0.1, f_inc=0.04, seed=7)
            ms_f, fl_f, out_f = timed(ctx, stream, lambda: P.round_adaptive_krp(y, c), 3)
            ctx.reset_counters()
            P.round_sum_adaptive_krp(terms, 1e-6, 0.04, 7)
            sk_sum = ctx.counters().sketch
            ctx.reset_counters()
            P.round_adaptive_krp(y, c)
            sk_formal = ctx.counters().sketch
            rec = dict(config="4sum: config 4 as 20 terms, adaptive tol 1e-6", ms_sum=ms_s, ranks_sum=out_s.ranks(),
                       ms_formal=ms_f, ranks_formal=out_f.ranks(), sketch_flops_sum=sk_sum,
                       sketch_flops_formal=sk_formal, rel_diff=P.relative_error(out_f, out_s))
        else:
            continue
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
