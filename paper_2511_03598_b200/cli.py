"""Command-line drop-in for the reference CLI's `round` command
(tools/ttround_main.cpp:86-184): round a TTF1 file on the B200 and print the
same JSON record (algorithm, mode, target, rel_error, ranks, wall_seconds,
flops_total/gemm/qr/svd/sketch, rng_draws, seed).

    python -m paper_2511_03598_b200.cli round IN.ttf1 OUT.ttf1 --algo krp-fix --ranks 10 10 10 --seed 7
    python -m paper_2511_03598_b200.cli round IN.ttf1 OUT.ttf1 --algo krp-adapt-r --tol 1e-6

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
    args = ap.parse_args(argv)
    try:
        return cmd_round(args)
    except TTRoundError as e:
        print(f"ttround error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
