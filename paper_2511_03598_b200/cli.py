"""Command-line drop-in for the reference CLI's `round` and `bench-synthetic`
commands (tools/ttround_main.cpp:86-210): round a TTF1 file on the B200 and
print the same JSON record (algorithm, mode, target, rel_error, ranks,
wall_seconds, flops_total/gemm/qr/svd/sketch, rng_draws, seed), or sweep the
synthetic benchmark into the same CSV schema.

    python -m paper_2511_03598_b200.cli round IN.ttf1 OUT.ttf1 --algo krp-fix --ranks 10 10 10 --seed 7
    python -m paper_2511_03598_b200.cli round IN.ttf1 OUT.ttf1 --algo krp-adapt-r --tol 1e-6
    python -m paper_2511_03598_b200.cli bench-synthetic --d 5 --n 20 --rank 10 --targets 10,12 --tols 1e-4 --csv b.csv

Algorithms: det, krp-fix, rand-orth, krp-adapt, krp-adapt-r (dispatch_rounding,
ttround_main.cpp:86-119). `--rng xoshiro` (default) reproduces the reference's
Gaussian stream and draw order; `--rng philox` draws the factors on the device.
Errors print `ttround error: <Errc>: <message>` and exit 2, as the reference.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

from . import (AdaptiveConfig, Context, RNG_PHILOX, RNG_XOSHIRO, TTRoundError, TTTensor, compression_pass,
               relative_error, round_adaptive_krp, round_deterministic, round_fixed_krp, round_rand_orth_tt)


def dispatch_rounding(algo, x, targets, tol, seed, rng):  # ttround_main.cpp:86-119
    if algo == "det":
        return round_deterministic(x, target_ranks=targets) if targets else round_deterministic(x, eps=tol)
    if algo == "krp-fix":
        if not targets:
            raise TTRoundError(10, "InvalidRanks: krp-fix requires --ranks")
        return round_fixed_krp(x, targets, seed, rng=rng)
    if algo == "rand-orth":
        if not targets:
            raise TTRoundError(10, "InvalidRanks: rand-orth requires --ranks")
        return round_rand_orth_tt(x, targets, seed, rng=rng)
    if algo in ("krp-adapt", "krp-adapt-r"):
        if tol is None:
            raise TTRoundError(14, "InvalidArgument: krp-adapt requires --tol")
        out = round_adaptive_krp(x, AdaptiveConfig(tolerance=tol, seed=seed, rng=rng))
        d = len(out.ranks()) - 1
        if algo == "krp-adapt-r" and d > 1:
            last = out.cores()[-1]
            nrm = float((last ** 2).sum()) ** 0.5
            out = compression_pass(out, tol * nrm / math.sqrt(d - 1))
        return out
    raise TTRoundError(14, f"InvalidArgument: unknown algorithm: {algo}")


def cmd_round(args) -> int:  # ttround_main.cpp:142-184
    ctx = Context(args.device)
    x = TTTensor.read_ttf1(args.input, ctx)
    d = len(x.ranks()) - 1
    targets = list(args.ranks) if args.ranks else None
    if targets is not None and len(targets) != d - 1:
        raise TTRoundError(10, f"InvalidRanks: expected {d - 1} target ranks, got {len(targets)}")
    if targets is None and args.tol is None:
        raise TTRoundError(14, "InvalidArgument: need --ranks or --tol")
    rng = RNG_XOSHIRO if args.rng == "xoshiro" else RNG_PHILOX
    ctx.reset_counters()
    ctx.synchronize()
    t0 = time.perf_counter()
    y = dispatch_rounding(args.algo, x, targets, args.tol, args.seed, rng)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    cnt = ctx.counters()
    y.write_ttf1(args.output)
    rec = {"algorithm": args.algo, "mode": "ranks" if targets else "tolerance",
           "target": float(max(targets)) if targets else args.tol, "rel_error": relative_error(x, y),
           "ranks": y.ranks(), "wall_seconds": wall, "flops_total": cnt.total(), "flops_gemm": cnt.gemm,
           "flops_qr": cnt.qr, "flops_svd": cnt.svd, "flops_sketch": cnt.sketch, "rng_draws": cnt.rng,
           "seed": args.seed}
    print(json.dumps(rec))
    return 0


BENCH_CSV_HEADER = ("algorithm,mode,target,rel_error,ranks,wall_seconds,flops_total,flops_gemm,flops_qr,"
                    "flops_svd,flops_sketch,rng_draws,seed")  # ttround_main.cpp:75-77


def fmt17(v: float) -> str:  # ttround_main.cpp:33-37
    return "%.17g" % v


def run_rounding(ctx, algo, x, targets, tol, seed, rng):  # ttround_main.cpp:121-140
    ctx.reset_counters()
    ctx.synchronize()
    t0 = time.perf_counter()
    y = dispatch_rounding(algo, x, targets, tol, seed, rng)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    cnt = ctx.counters()
    return {"algorithm": algo, "mode": "ranks" if targets else "tolerance",
            "target": float(max(targets)) if targets else tol, "rel_error": relative_error(x, y),
            "ranks": y.ranks(), "wall_seconds": wall, "counts": cnt, "seed": seed}


def csv_row(r) -> str:  # ttround_main.cpp:79-84
    c = r["counts"]
    return ",".join([r["algorithm"], r["mode"], fmt17(r["target"]), fmt17(r["rel_error"]),
                     "x".join(str(v) for v in r["ranks"]), fmt17(r["wall_seconds"]), str(c.total()), str(c.gemm),
                     str(c.qr), str(c.svd), str(c.sketch), str(c.rng), str(r["seed"])])


def synthetic_perturbed_tt(ctx, d, n, r, eps, seed):
    """synthetic.cpp:8-26 on the device: Y, Z Gaussian TTs (reference stream, shared rank
    chain) normalised by norm_exact, X = formal_sum(Y, eps Z)."""
    from . import formal_sum, norm_exact, scaled
    from .seeds import derive_seed
    ranks = [1] + [r] * (d - 1) + [1]
    y = TTTensor.random_gaussian([n] * d, ranks, derive_seed(seed, 1), ctx)
    z = TTTensor.random_gaussian([n] * d, ranks, derive_seed(seed, 2), ctx)
    y = scaled(y, 1.0 / norm_exact(y))
    z = scaled(z, 1.0 / norm_exact(z))
    return formal_sum([y, scaled(z, eps)])


# Orth-Rand (round_orth_rand, round_rand.cpp:181-240) is outside this repo's
# scope: its rows are not produced.
OMITTED = ["orth-rand"]


def cmd_bench_synthetic(args) -> int:  # ttround_main.cpp:178-210
    d, n, rank, eps, seeds = args.d, args.n, args.rank, args.eps_pert, args.seeds
    if d < 2 or n < 1 or rank < 1 or eps < 0 or seeds < 1:
        raise TTRoundError(14, "InvalidArgument: invalid benchmark parameters")
    targets = [int(v) for v in args.targets.split(",")] if args.targets else []
    tols = [float(v) for v in args.tols.split(",")] if args.tols else []
    if not targets and not tols:
        raise TTRoundError(14, "InvalidArgument: need --targets or --tols")
    ctx = Context(args.device)
    x = synthetic_perturbed_tt(ctx, d, n, rank, eps, args.master_seed)
    rng = RNG_XOSHIRO if args.rng == "xoshiro" else RNG_PHILOX
    try:
        f = open(args.csv, "w")
    except OSError:
        raise TTRoundError(15, f"IoError: cannot open {args.csv}")
    with f:
        f.write(BENCH_CSV_HEADER + "\n")
        for target in targets:
            tr = [target] * (d - 1)
            for seed in range(seeds):
                for algo in ("det", "krp-fix", "rand-orth"):
                    f.write(csv_row(run_rounding(ctx, algo, x, tr, None, seed, rng)) + "\n")
        for tol in tols:
            for seed in range(seeds):
                for algo in ("det", "krp-adapt", "krp-adapt-r"):
                    f.write(csv_row(run_rounding(ctx, algo, x, None, tol, seed, rng)) + "\n")
    print(json.dumps({"csv": args.csv, "d": d, "n": n, "rank": rank, "eps_pert": eps, "x_ranks": x.ranks(),
                      "omitted_algorithms": OMITTED}))
    return 0


COOKIE_STRATEGIES = {"det": 0, "rand-orth": 1, "krp-adapt-sum": 2}


def cmd_cookie(args) -> int:  # ttround_main.cpp:246-296
    import paper_2511_03598_b200 as P
    ctx = P.Context(args.device)
    op, rhs = P.cookie_problem(args.params, args.grid, args.nsamples, args.rho_min, args.rho_max, ctx)
    track = not args.no_true_residual
    res = P.tt_gmres(op, rhs, rel_tolerance=args.tol, max_iterations=args.max_iters,
                     strategy=COOKIE_STRATEGIES[args.strategy], rounding_tolerance=args.round_tol, seed=args.seed,
                     track_true_residual=track, rng=P.RNG_XOSHIRO if args.rng == "xoshiro" else P.RNG_PHILOX)
    if args.csv:
        try:
            with open(args.csv, "w") as f:
                f.write("iteration,rel_residual,max_tt_rank,cum_rounding_seconds\n")
                for i in range(res["iterations"]):
                    resid = res["true_residual_history"][i] if track else res["residual_history"][i]
                    f.write(f"{i + 1},{fmt17(resid)},{res['max_rank_history'][i]},"
                            f"{fmt17(res['rounding_seconds_history'][i])}\n")
        except OSError:
            raise TTRoundError(15, f"IoError: cannot open {args.csv}")
    summary = {"converged": res["converged"], "iterations": res["iterations"], "strategy": args.strategy,
               "arnoldi_residual": res["residual_history"][-1] if res["residual_history"] else 0.0,
               "solution_ranks": res["solution"].ranks(), "rounding_seconds": res["rounding_seconds"],
               "seed": args.seed}
    if track and res["true_residual_history"]:
        summary["true_residual"] = res["true_residual_history"][-1]
    if args.csv:
        summary["csv"] = args.csv
    print(json.dumps(summary))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ttround-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("round", help="round a TTF1 file")
    r.add_argument("input")
    r.add_argument("output")
    r.add_argument("--algo", default="krp-fix", choices=["det", "krp-fix", "rand-orth", "krp-adapt", "krp-adapt-r"])
    r.add_argument("--ranks", type=int, nargs="*")
    r.add_argument("--tol", type=float)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--rng", default="xoshiro", choices=["xoshiro", "philox"])
    r.add_argument("--device", type=int, default=0)
    b = sub.add_parser("bench-synthetic", help="rounding benchmark on perturbed low-rank tensors")
    b.add_argument("--d", type=int, default=5)
    b.add_argument("--n", type=int, default=20)
    b.add_argument("--rank", type=int, default=10)
    b.add_argument("--eps-pert", type=float, default=1e-5)
    b.add_argument("--targets", default="")
    b.add_argument("--tols", default="")
    b.add_argument("--seeds", type=int, default=10)
    b.add_argument("--csv", default="bench.csv")
    b.add_argument("--master-seed", type=int, default=20250807)
    b.add_argument("--rng", default="xoshiro", choices=["xoshiro", "philox"])
    b.add_argument("--device", type=int, default=0)
    k = sub.add_parser("cookie", help="parametric cookie problem via TT-GMRES")
    k.add_argument("--params", type=int, default=3)
    k.add_argument("--grid", type=int, default=16)
    k.add_argument("--nsamples", type=int, default=8)
    k.add_argument("--rho-min", type=float, default=1.0)
    k.add_argument("--rho-max", type=float, default=10.0)
    k.add_argument("--tol", type=float, default=1e-6)
    k.add_argument("--strategy", default="krp-adapt-sum", choices=list(COOKIE_STRATEGIES))
    k.add_argument("--seed", type=int, default=0)
    k.add_argument("--csv", default="")
    k.add_argument("--max-iters", type=int, default=250)
    k.add_argument("--round-tol", type=float, default=0.0)
    k.add_argument("--no-true-residual", action="store_true")
    k.add_argument("--rng", default="xoshiro", choices=["xoshiro", "philox"])
    k.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "bench-synthetic":
            return cmd_bench_synthetic(args)
        if args.cmd == "cookie":
            return cmd_cookie(args)
        return cmd_round(args)
    except TTRoundError as e:
        print(f"ttround error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
