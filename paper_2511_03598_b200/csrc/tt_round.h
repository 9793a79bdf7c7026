// tt_round.h — device-resident TT container and the rounding entry points
// (host orchestration in tt_round.cu / tt_det.cu).
#pragma once

#include <algorithm>
#include <functional>
#include <memory>
#include <vector>

#include "common.cuh"

namespace ttr {

// Device TT tensor: all cores in one allocation, each 256-byte aligned, in
// the reference layout (core k = column-major vertical unfolding of the
// r_{k-1} x n_k x r_k core, proj/core/include/ttround/tensor.hpp:11-16).
struct TTDev {
    Ctx* ctx;
    std::vector<i64> n, r, off;
    DBuf buf;
    TTDev(Ctx& c, const std::vector<i64>& n, const std::vector<i64>& r);
    i64 d() const { return static_cast<i64>(n.size()); }
    double* core(i64 k) const { return buf.p + off[k]; }
    i64 core_size(i64 k) const { return r[k] * n[k] * r[k + 1]; }
    i64 total() const;
    i64 max_rank() const;
    void upload(const double* host);
    void download(double* host) const;
};

// Batch of identically shaped TT tensors: tensor b occupies
// [b*stride, (b+1)*stride) of one allocation, cores laid out as in TTDev.
struct TTBatch {
    Ctx* ctx;
    std::vector<i64> n, r, off;
    i64 stride = 0, batch = 0;
    DBuf buf;
    TTBatch(Ctx& c, i64 batch, const std::vector<i64>& n, const std::vector<i64>& r);
    i64 d() const { return static_cast<i64>(n.size()); }
    double* core(i64 b, i64 k) const { return buf.p + b * stride + off[k]; }
    i64 core_size(i64 k) const { return r[k] * n[k] * r[k + 1]; }
    i64 total() const;
    i64 max_rank() const { return *std::max_element(r.begin(), r.end()); }
};
std::unique_ptr<TTBatch> batch_two_part_philox(Ctx& c, i64 batch, i64 d, i64 n, i64 rx, i64 rz, double eps,
                                               std::uint64_t seed);
std::unique_ptr<TTBatch> round_fixed_krp_batched(Ctx& c, const TTBatch& t, const std::vector<i64>& targets,
                                                 std::uint64_t seed);

struct AdaptiveCfg {
    double tolerance = 1e-6, f_init = 0.1, f_inc = 0.05;
    std::uint64_t seed = 0;
    bool has_known_norm = false;
    double known_norm = 0.0;
    const i64* max_rank_cap = nullptr;
    int rng_mode = TTR_RNG_PHILOX;
};

std::unique_ptr<TTDev> copy_tt(Ctx& c, const TTDev& t);
// TTTensor constructor's finiteness scan (tensor.cpp:75-78): InvalidArgument
// "core entries must be finite" on any NaN/Inf core entry.
void check_finite(Ctx& c, const TTDev& t);
// dot (tensor.cpp:244-256): <a, b> by the core-contraction sweep (DMMA GEMMs).
double dot(Ctx& c, const TTDev& a, const TTDev& b);
// random_gaussian_tt (tensor.cpp:217-242) from the reference's xoshiro stream
// (host draws, bitwise the reference), uploaded.
std::unique_ptr<TTDev> random_gaussian_tt(Ctx& c, const std::vector<i64>& n, const std::vector<i64>& r,
                                          std::uint64_t seed);
std::unique_ptr<TTDev> random_philox_tt(Ctx& c, const std::vector<i64>& n, const std::vector<i64>& r, std::uint64_t seed);
std::unique_ptr<TTDev> formal_sum(Ctx& c, const std::vector<const TTDev*>& terms);
std::unique_ptr<TTDev> kernel_sum_tt(Ctx& c, i64 d, i64 n, i64 r, i64 terms, double ell, std::uint64_t seed);
std::unique_ptr<TTDev> kernel_term_tt(Ctx& c, i64 d, i64 n, i64 r, i64 t, double ell, std::uint64_t seed);
void scale_tt(Ctx& c, TTDev& t, double alpha);
std::unique_ptr<TTDev> orthogonalize_rl_public(Ctx& c, const TTDev& t);
double norm_exact(Ctx& c, const TTDev& t);
double relative_error(Ctx& c, const TTDev& a, const TTDev& b);

std::unique_ptr<TTDev> round_fixed_krp(Ctx& c, const TTDev& t, const std::vector<i64>& target_ranks, std::uint64_t seed,
                                       int rng_mode);
std::vector<i64> fixed_krp_ranks(const TTDev& t, const std::vector<i64>& target_ranks);
void round_fixed_krp_into(Ctx& c, const TTDev& t, const std::vector<i64>& target_ranks, std::uint64_t seed,
                          int rng_mode, TTDev& out);
// Runs a rounding whose sweep may take the Cholesky QR, then checks the
// breakdown flag once and reruns it on the Householder path if set.
void with_qr_speculation(Ctx& c, const std::function<void()>& body);
void rand_orth_sweep(Ctx& c, const TTDev& t, i64 width, const std::vector<const double*>& W,
                     const std::vector<i64>& ldw, TTDev& out);
void krp_sketch_into(Ctx& c, const TTDev& t, i64 col0, i64 ncols, std::uint64_t seed, const std::vector<double*>& W,
                     const std::vector<i64>& ldw);

// Captured CUDA graph of round_fixed_krp for a fixed input buffer (contents
// may change between executions) writing into an owned output tensor.
struct Plan {
    Ctx& c;
    const TTDev& in;
    std::vector<i64> ranks;
    std::uint64_t seed;
    int rng_mode;
    const double* host_in = nullptr;
    double* host_out = nullptr;
    std::unique_ptr<TTDev> out;  // moved to the C handle after construction
    TTDev* target = nullptr;     // the output tensor every graph writes
    cudaGraph_t graph = nullptr, graph_safe = nullptr;
    cudaGraphExec_t exec = nullptr, exec_safe = nullptr;  // speculative (Cholesky QR) / Householder
    bool speculative = false;
    i64 hh_from = INT32_MAX;  // modes >= hh_from take the Householder QR in the speculative graph
    std::uint64_t launches_per_run = 0;
    Counts flops;
    HostIO io;  // host-streaming plans only
    cudaEvent_t fork = nullptr, join = nullptr;
    // host_in/host_out (pinned, flat cores): the graph also streams the input
    // in and the result out, overlapped with the sweep
    Plan(Ctx& c, const TTDev& in, const std::vector<i64>& ranks, std::uint64_t seed, int rng_mode,
         const double* host_in = nullptr, double* host_out = nullptr);
    ~Plan();
    bool capture(bool spec, cudaGraph_t& g, cudaGraphExec_t& e);
    void execute();
};

std::unique_ptr<TTDev> round_adaptive_krp(Ctx& c, const TTDev& t, const AdaptiveCfg& cfg, std::vector<double>* trace);

// Growth decisions of one adaptive round: recorded by an eager run, replayed
// (and verified on the device) by a captured one (AdaptivePlan).
struct AdaptiveTape {
    bool replay = false;
    std::vector<char> stops;  // one per growth test: 1 = the residual estimate met tau
    std::size_t pos = 0;
    double* d_tau = nullptr;
    double* d_scratch = nullptr;  // [2]
    int* d_mismatch = nullptr;
};
// round_adaptive_krp with an optional decision tape and output tensor (the
// plan's replay writes into the recorded run's output; returns null then)
std::unique_ptr<TTDev> round_adaptive_krp_impl(Ctx& c, const TTDev& t, const AdaptiveCfg& cfg,
                                               std::vector<double>* trace, AdaptiveTape* tape, TTDev* out_into);
struct AdaptivePlan {
    Ctx& c;
    const TTDev& in;
    AdaptiveCfg cfg;
    std::vector<i64> caps;
    std::unique_ptr<TTDev>* out_slot;  // the caller-visible output (replaced when the plan re-records)
    AdaptiveTape tape;
    Ctx::QrTape qr_tape;  // which growth/initial QRs took the Householder panels (checked Cholesky-QR, qr.cu)
    DBuf dev;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::uint64_t launches_per_run = 0;
    Counts flops;
    bool counted = false;
    int rerecords = 0;
    AdaptivePlan(Ctx& c, const TTDev& in, const AdaptiveCfg& cfg, std::unique_ptr<TTDev>* out_slot);
    ~AdaptivePlan();
    void rebuild();
    void execute();
};
// round_rand.cpp:66-78 — Rand-Orth with a Gaussian TT sketch (reference xoshiro stream for R)
std::unique_ptr<TTDev> round_rand_orth_tt(Ctx& c, const TTDev& t, const std::vector<i64>& target_ranks,
                                          std::uint64_t seed, int rng_mode);
// adaptive growth step: Qb(:, q:q+grow) = orthonormal basis of the projected
// sketch block Sb (rows x grow, ld rows); Qn/P scratch (tt_round.cu)
void growth_basis(Ctx& c, i64 rows, i64 q, i64 grow, double* Qb, double* Sb, double* Qn, double* P);
// sum_round.cpp:52-173 — adaptive rounding of sum(terms) without the formal sum (tt_sum.cu)
std::unique_ptr<TTDev> round_sum_adaptive_krp(Ctx& c, const std::vector<const TTDev*>& terms, double eps, double f_inc,
                                              std::uint64_t seed, int rng_mode);
double estimate_norm_krp(Ctx& c, const TTDev& t, i64 width, std::uint64_t seed, int rng_mode);
std::unique_ptr<TTDev> round_deterministic_tol(Ctx& c, const TTDev& t, double eps);
// round_rand.cpp:155-179 — right-to-left truncation pass of a left-orthogonal TT (tt_det.cu)
std::unique_ptr<TTDev> compression_pass(Ctx& c, const TTDev& left_orthogonal, double tau);
std::unique_ptr<TTDev> round_deterministic_ranks(Ctx& c, const TTDev& t, const std::vector<i64>& ranks);

// W_start..W_d of the KRP partial contractions for explicit (or Philox) factors.
void krp_partial_contractions(Ctx& c, const TTDev& t, i64 start_mode, i64 cols, const double* host_factors,
                              std::uint64_t seed, i64 col0, double* host_w);

}  // namespace ttr

struct ttr_tt {
    std::unique_ptr<ttr::TTDev> t;
};
struct ttr_ctx {
    ttr::Ctx c;
};
struct ttr_batch {
    std::unique_ptr<ttr::TTBatch> t;
};
struct ttr_plan {
    std::unique_ptr<ttr::Plan> plan;
    std::unique_ptr<ttr::AdaptivePlan> aplan;
    ttr_tt out;
    ttr_ctx* ctx = nullptr;
};
