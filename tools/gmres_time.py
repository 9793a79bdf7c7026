"""The reference's acceptance criterion 8 (TT-GMRES on build_cookie_problem(3, 16,
8, 1, 10), tol 1e-6, deterministic + AdaptiveKRPSum seeds 1-3, reference xoshiro
sketches) through the device harness, with the CPU oracle's run of the same
four solves timed beside it (host wall clock). Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2511_03598_b200 as P  # noqa: E402
import py_oracle as O  # noqa: E402


def main():
    op, rhs = P.cookie_problem(3, 16, 8, 1.0, 10.0)
    kw = dict(rel_tolerance=1e-6, max_iterations=250, track_true_residual=False)
    P.tt_gmres(op, rhs, strategy=P.GMRES_DETERMINISTIC, **kw)  # warm-up (pools, kernels)
    runs = []
    t0 = time.perf_counter()
    det = P.tt_gmres(op, rhs, strategy=P.GMRES_DETERMINISTIC, **kw)
    runs.append(("det", 0, det))
    for seed in (1, 2, 3):
        runs.append(("krp-adapt-sum", seed, P.tt_gmres(op, rhs, strategy=P.GMRES_ADAPTIVE_KRP_SUM, seed=seed,
                                                        rng=P.RNG_XOSHIRO, **kw)))
    gpu_s = time.perf_counter() - t0
    rec = {"workload": "acceptance criterion 8: tt_gmres(cookie(3,16,8,1,10)), tol 1e-6, det + krp-adapt-sum x3",
           "gpu_seconds_total": gpu_s,
           "runs": [{"strategy": s, "seed": sd, "iterations": r["iterations"], "converged": r["converged"],
                     "arnoldi_residual": r["residual_history"][-1], "rounding_seconds": r["rounding_seconds"]}
                    for s, sd, r in runs]}
    if "--cpu" in sys.argv:
        t0 = time.perf_counter()
        O.tt_gmres_cookie(3, 16, 8, 1.0, 10.0, rel_tolerance=1e-6, max_iterations=250, strategy=O.DETERMINISTIC,
                          track_true_residual=False)
        for seed in (1, 2, 3):
            O.tt_gmres_cookie(3, 16, 8, 1.0, 10.0, rel_tolerance=1e-6, max_iterations=250,
                              strategy=O.ADAPTIVE_KRP_SUM, seed=seed, track_true_residual=False)
        rec["cpu_seconds_total"] = time.perf_counter() - t0
        rec["cpu_kind"] = "oracle restatement of solver.cpp (port backend), host wall clock"
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
