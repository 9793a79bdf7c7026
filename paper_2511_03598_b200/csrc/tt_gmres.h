// tt_gmres.h — device TT-GMRES cookie harness (tt_gmres.cu; solver.hpp).
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"
#include "tt_round.h"

namespace ttr {

// KroneckerSumOperator (solver.hpp:12-21): nterms terms of d square factors.
// factors: term-major, then mode, each n_k x n_k column-major.
struct KronOpDev {
    std::vector<i64> n;
    i64 nterms = 0;
    std::vector<std::vector<DBuf>> At;                  // A_{i,k}^T on the device
    std::vector<std::vector<std::vector<double>>> host; // A_{i,k} (host copy: mean-field matrix)
    std::vector<std::vector<bool>> identity;            // A_{i,k} == I (copied, not multiplied)
    KronOpDev(Ctx& c, i64 nterms, const std::vector<i64>& n, const double* factors);
};

struct GmresResultDev {
    std::unique_ptr<TTDev> solution;
    std::vector<double> residual_history, true_residual_history, rounding_seconds_history;
    std::vector<i64> max_rank_history;
    double rounding_seconds = 0.0;
    i64 iterations = 0;
    bool converged = false;
};

std::unique_ptr<KronOpDev> cookie_problem(Ctx& c, i64 p, i64 grid, i64 samples, double rho_min, double rho_max,
                                          std::unique_ptr<TTDev>* rhs);
std::vector<std::unique_ptr<TTDev>> apply_operator(Ctx& c, const KronOpDev& op, const TTDev& x);
GmresResultDev tt_gmres(Ctx& c, const KronOpDev& op, const TTDev& rhs, const ttr_gmres_cfg& cfg);

}  // namespace ttr

struct ttr_kron_op {
    std::unique_ptr<ttr::KronOpDev> op;
};
