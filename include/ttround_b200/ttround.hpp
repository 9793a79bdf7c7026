// ttround.hpp — header-only C++ drop-in for the reference `ttround` hot path,
// implemented on top of the C ABI of libttround_b200 (include/ttround_b200.h).
//
// Mirrors the reference declarations a caller of the rounding path uses
// (proj/core/include/ttround/{types,tensor,round_rand,orthogonalize,sketch,flops}.hpp):
//
//   ttround::Errc / Error / fail            types.hpp:15-63
//   ttround::TTTensor (device resident)     tensor.hpp:124-149
//   round_fixed_krp                         round_rand.hpp:14-15
//   AdaptiveConfig / round_adaptive_krp     round_rand.hpp:18-31
//   TTSum / round_sum_adaptive_krp          sum_round.hpp:11-29
//   KroneckerSumOperator / build_cookie_problem / apply_operator / tt_gmres   solver.hpp:12-82
//   round_deterministic (tolerance / ranks) orthogonalize.hpp:50,54
//   estimate_norm_krp                       sketch.hpp:63
//   norm_exact / relative_error / formal_sum / scaled   tensor.hpp:172-191
//   flops::counters / reset                 flops.hpp:12-25
//   Core / TTTensor(std::vector<Core>)      tensor.hpp:17-63
//   random_gaussian_tt / dot                tensor.hpp:111,119
//   GaussianStream                          rng.hpp:12-35
//   GaussianFactorSet / draw_gaussian_factors / append_gaussian_columns   sketch.hpp:13-29
//   PartialContractionSet / krp_partial_contractions_rl / append_krp_contractions   sketch.hpp:35-53
//   generate_residual_sketch                round_rand.hpp:37-39
//   residual_norm_estimate                  sketch.hpp:67
//
// Differences a caller sees: cores live in HBM (construct from host cores,
// read back with cores()); every call takes an optional Context (default: a
// per-thread context on device 0); matrices are the small column-major
// ttround::Matrix below instead of Eigen::MatrixXd. The sketch generator
// defaults to RngMode::Xoshiro, the reference's own sequential stream, so a
// drop-in call round_fixed_krp(x, ranks, seed) draws exactly the reference's
// Omega; RngMode::Philox selects the counter-based device generator (no host
// draws; required by the CUDA-graph plans). Errors are rethrown as
// ttround::Error with the same Errc kinds the reference uses; failures of the
// device itself (CUDA, out of memory, NCCL, no device) are ttround::DeviceError
// (Errc::DeviceFailure, a kind the reference does not have).
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ttround_b200.h"

namespace ttround {

using Index = std::int64_t;

enum class Errc {
    RankChainMismatch, BoundaryRankNotOne, EmptyCoreList, IndexOutOfRange, DenseTooLarge,
    ModeSizeMismatch, EmptyTermList, InvalidRankChain, SVDFailure, InvalidRanks,
    NotLeftOrthogonal, InvalidGrid, Breakdown, InvalidArgument, IoError,
    DeviceFailure,  // not in the reference: CUDA / out-of-memory / NCCL / no-device failures
};

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& what, int status = 0)
        : std::runtime_error(what), code_(code), status_(status) {}
    Errc code() const noexcept { return code_; }
    int status() const noexcept { return status_; }  // raw ttr_status (>= 100: device failure)

private:
    Errc code_;
    int status_;
};

//! A failure of the device rather than of the caller's input: status() is the
//! raw ttr_status (TTR_ERR_CUDA, _OUT_OF_MEMORY, _NCCL, _INTERNAL, _NO_DEVICE).
class DeviceError : public Error {
public:
    DeviceError(const std::string& what, int status) : Error(Errc::DeviceFailure, what, status) {}
    bool out_of_memory() const noexcept { return status() == TTR_ERR_OUT_OF_MEMORY; }
};

[[noreturn]] inline void fail(Errc code, const std::string& what) { throw Error(code, what); }

inline void check(ttr_status s) {
    if (s == TTR_OK) return;
    const std::string msg = ttr_last_error();
    if (s >= 1 && s <= 15) throw Error(static_cast<Errc>(s - 1), msg, s);
    throw DeviceError(msg, s);
}

enum class RngMode : int { Xoshiro = TTR_RNG_XOSHIRO, Philox = TTR_RNG_PHILOX };

//! Column-major dense matrix (the reference's Eigen::MatrixXd at this boundary).
struct Matrix {
    Index rows_ = 0, cols_ = 0;
    std::vector<double> a;
    Matrix() = default;
    Matrix(Index r, Index c) : rows_(r), cols_(c), a(static_cast<std::size_t>(r * c), 0.0) {}
    Index rows() const noexcept { return rows_; }
    Index cols() const noexcept { return cols_; }
    double& operator()(Index i, Index j) { return a[static_cast<std::size_t>(i + j * rows_)]; }
    double operator()(Index i, Index j) const { return a[static_cast<std::size_t>(i + j * rows_)]; }
    double* data() noexcept { return a.data(); }
    const double* data() const noexcept { return a.data(); }
};

//! A 3-way TT core r_left x n x r_right on the host, stored as the column-major
//! vertical unfolding: element (i, j, g) at g*r_left*n + j*r_left + i
//! (tensor.hpp:11-54). The TTTensor built from cores lives on the device.
class Core {
public:
    Core(Index r_left, Index n, Index r_right)
        : rl_(r_left), n_(n), rr_(r_right), data_(checked(r_left, n, r_right), 0.0) {}
    Core(Index r_left, Index n, Index r_right, std::vector<double> entries)
        : rl_(r_left), n_(n), rr_(r_right), data_(std::move(entries)) {
        if (static_cast<Index>(data_.size()) != static_cast<Index>(checked(r_left, n, r_right)))
            fail(Errc::InvalidArgument, "core entry count does not match shape");
    }
    static Core from_vertical(Index r_left, Index n, const Matrix& v) {
        if (v.rows() != r_left * n) fail(Errc::InvalidArgument, "vertical unfolding shape mismatch");
        return Core(r_left, n, v.cols(), v.a);
    }
    static Core from_horizontal(Index n, Index r_right, const Matrix& h) {
        if (h.cols() != n * r_right) fail(Errc::InvalidArgument, "horizontal unfolding shape mismatch");
        return Core(h.rows(), n, r_right, h.a);
    }
    Index r_left() const noexcept { return rl_; }
    Index n() const noexcept { return n_; }
    Index r_right() const noexcept { return rr_; }
    Index size() const noexcept { return static_cast<Index>(data_.size()); }
    double operator()(Index i, Index j, Index g) const { return data_[static_cast<std::size_t>(g * rl_ * n_ + j * rl_ + i)]; }
    double& operator()(Index i, Index j, Index g) { return data_[static_cast<std::size_t>(g * rl_ * n_ + j * rl_ + i)]; }
    const std::vector<double>& data() const noexcept { return data_; }
    std::vector<double>& data() noexcept { return data_; }

private:
    static std::size_t checked(Index rl, Index n, Index rr) {
        if (rl < 1 || n < 1 || rr < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
        return static_cast<std::size_t>(rl * n * rr);
    }
    Index rl_, n_, rr_;
    std::vector<double> data_;
};

class Context {
public:
    explicit Context(int device = 0, void* cuda_stream = nullptr) { check(ttr_ctx_create(device, cuda_stream, &h_)); }
    ~Context() { ttr_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ttr_ctx* get() const { return h_; }
    void synchronize() const { check(ttr_ctx_synchronize(h_)); }
    static Context& thread_default() {
        thread_local Context ctx(0);
        return ctx;
    }

private:
    ttr_ctx* h_ = nullptr;
};

//! Device-resident TT tensor (reference layout: core k = column-major vertical
//! unfolding of the r_{k-1} x n_k x r_k core, tensor.hpp:11-16).
class TTTensor {
public:
    TTTensor(const std::vector<Index>& mode_sizes, const std::vector<Index>& ranks,
             const std::vector<double>& cores_concat, Context& ctx = Context::thread_default())
        : ctx_(&ctx) {
        ttr_tt* t = nullptr;
        check(ttr_tt_upload(ctx.get(), static_cast<int64_t>(mode_sizes.size()), mode_sizes.data(), ranks.data(),
                            cores_concat.data(), &t));
        h_.reset(t, &ttr_tt_destroy);
    }
    //! TTTensor(std::vector<Core>) (tensor.hpp:63): the constructor's checks
    //! (tensor.cpp:66-79, incl. the finiteness scan, run on the device).
    explicit TTTensor(const std::vector<Core>& cores, Context& ctx = Context::thread_default()) : ctx_(&ctx) {
        std::vector<int64_t> rl, n, rr;
        std::vector<const double*> ptrs;
        for (const auto& c : cores) {
            rl.push_back(c.r_left());
            n.push_back(c.n());
            rr.push_back(c.r_right());
            ptrs.push_back(c.data().data());
        }
        ttr_tt* t = nullptr;
        check(ttr_tt_upload_cores(ctx.get(), static_cast<int64_t>(cores.size()), rl.data(), n.data(), rr.data(),
                                  ptrs.data(), &t));
        h_.reset(t, &ttr_tt_destroy);
    }
    TTTensor(ttr_tt* owned, Context& ctx) : h_(owned, &ttr_tt_destroy), ctx_(&ctx) {}

    Index order() const { return static_cast<Index>(mode_sizes().size()); }
    std::vector<Index> mode_sizes() const {
        int64_t d = 0;
        check(ttr_tt_shape(h_.get(), &d, nullptr, nullptr, nullptr));
        std::vector<Index> n(static_cast<std::size_t>(d));
        check(ttr_tt_shape(h_.get(), &d, n.data(), nullptr, nullptr));
        return n;
    }
    std::vector<Index> ranks() const {
        int64_t d = 0;
        check(ttr_tt_shape(h_.get(), &d, nullptr, nullptr, nullptr));
        std::vector<Index> r(static_cast<std::size_t>(d + 1));
        check(ttr_tt_shape(h_.get(), &d, nullptr, r.data(), nullptr));
        return r;
    }
    Index rank(Index k) const { return ranks()[static_cast<std::size_t>(k)]; }
    Index max_rank() const {
        Index m = 1;
        for (Index r : ranks()) m = r > m ? r : m;
        return m;
    }
    //! All cores, concatenated, copied to the host.
    std::vector<double> cores() const {
        int64_t d = 0, total = 0;
        check(ttr_tt_shape(h_.get(), &d, nullptr, nullptr, &total));
        std::vector<double> out(static_cast<std::size_t>(total));
        check(ttr_tt_download(ctx_->get(), h_.get(), out.data()));
        return out;
    }
    //! Core k copied to the host (Core(k) of the reference, tensor.hpp:70).
    Core core(Index k) const {
        const auto n = mode_sizes();
        const auto r = ranks();
        if (k < 0 || k >= static_cast<Index>(n.size())) fail(Errc::IndexOutOfRange, "core index out of range");
        std::vector<double> host(static_cast<std::size_t>(r[k] * n[k] * r[k + 1]));
        check(ttr_tt_download_core(ctx_->get(), h_.get(), k, host.data()));
        return Core(r[k], n[k], r[k + 1], std::move(host));
    }
    ttr_tt* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    std::shared_ptr<ttr_tt> h_;
    Context* ctx_;
};

struct AdaptiveConfig {  // round_rand.hpp:18-25
    double tolerance = 1e-6;
    double f_init = 0.1;
    double f_inc = 0.05;
    std::uint64_t seed = 0;
    std::optional<double> known_norm;
    std::optional<std::vector<Index>> max_rank_cap;
    RngMode rng = RngMode::Xoshiro;  // the reference's stream (Philox: device generator)
};

inline TTTensor round_fixed_krp(const TTTensor& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                                RngMode rng = RngMode::Xoshiro) {
    ttr_tt* out = nullptr;
    check(ttr_round_fixed_krp(tt.context().get(), tt.get(), target_ranks.data(),
                              static_cast<int64_t>(target_ranks.size()), seed, static_cast<int>(rng), &out));
    return TTTensor(out, tt.context());
}

inline TTTensor round_adaptive_krp(const TTTensor& tt, const AdaptiveConfig& cfg) {
    ttr_adaptive_cfg c{};
    c.tolerance = cfg.tolerance;
    c.f_init = cfg.f_init;
    c.f_inc = cfg.f_inc;
    c.seed = cfg.seed;
    c.has_known_norm = cfg.known_norm.has_value() ? 1 : 0;
    c.known_norm = cfg.known_norm.value_or(0.0);
    c.max_rank_cap = cfg.max_rank_cap ? cfg.max_rank_cap->data() : nullptr;
    c.max_rank_cap_len = cfg.max_rank_cap ? static_cast<int64_t>(cfg.max_rank_cap->size()) : 0;
    c.rng_mode = static_cast<int>(cfg.rng);
    ttr_tt* out = nullptr;
    check(ttr_round_adaptive_krp(tt.context().get(), tt.get(), &c, &out));
    return TTTensor(out, tt.context());
}

//! io.hpp: TTF1 files read straight into / written from a device tensor.
inline TTTensor read_ttf1(const std::string& path, Context& ctx = Context::thread_default()) {
    ttr_tt* out = nullptr;
    check(ttr_tt_read_ttf1(ctx.get(), path.c_str(), &out));
    return TTTensor(out, ctx);
}
inline void write_ttf1(const TTTensor& tt, const std::string& path) {
    check(ttr_tt_write_ttf1(tt.context().get(), tt.get(), path.c_str()));
}

//! round_rand.hpp:49 round_rand_orth_tt: Rand-Orth with a Gaussian TT sketch.
inline TTTensor round_rand_orth_tt(const TTTensor& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                                   RngMode rng = RngMode::Xoshiro) {
    ttr_tt* out = nullptr;
    check(ttr_round_rand_orth_tt(tt.context().get(), tt.get(), target_ranks.data(),
                                 static_cast<int64_t>(target_ranks.size()), seed, static_cast<int>(rng), &out));
    return TTTensor(out, tt.context());
}

//! round_rand.hpp compression_pass: right-to-left truncation of a left-orthogonal TT.
inline TTTensor compression_pass(const TTTensor& left_orthogonal, double tau) {
    ttr_tt* out = nullptr;
    check(ttr_compression_pass(left_orthogonal.context().get(), left_orthogonal.get(), tau, &out));
    return TTTensor(out, left_orthogonal.context());
}

//! A sum of TT tensors kept as its list of summands (sum_round.hpp:11-21).
struct TTSum {
    std::vector<TTTensor> terms;
    static TTSum of(std::vector<TTTensor> terms) {
        if (terms.empty()) throw Error(Errc::EmptyTermList, "sum of no TT terms");
        TTSum s;
        s.terms = std::move(terms);
        return s;
    }
};

//! Adaptive rounding of a sum without the formal sum (sum_round.hpp:29).
inline TTTensor round_sum_adaptive_krp(const TTSum& sum, double eps, double f_inc, std::uint64_t seed,
                                       RngMode rng = RngMode::Xoshiro) {
    std::vector<const ttr_tt*> hs;
    for (const auto& t : sum.terms) hs.push_back(t.get());
    ttr_tt* out = nullptr;
    Context& ctx = sum.terms.front().context();
    check(ttr_round_sum_adaptive_krp(ctx.get(), hs.data(), static_cast<int64_t>(hs.size()), eps, f_inc, seed,
                                     static_cast<int>(rng), &out));
    return TTTensor(out, ctx);
}

inline TTTensor round_deterministic(const TTTensor& tt, double eps) {
    ttr_tt* out = nullptr;
    check(ttr_round_deterministic_tol(tt.context().get(), tt.get(), eps, &out));
    return TTTensor(out, tt.context());
}

inline TTTensor round_deterministic(const TTTensor& tt, const std::vector<Index>& target_ranks) {
    ttr_tt* out = nullptr;
    check(ttr_round_deterministic_ranks(tt.context().get(), tt.get(), target_ranks.data(),
                                        static_cast<int64_t>(target_ranks.size()), &out));
    return TTTensor(out, tt.context());
}

inline double estimate_norm_krp(const TTTensor& tt, Index width, std::uint64_t seed, RngMode rng = RngMode::Xoshiro) {
    double v = 0.0;
    check(ttr_estimate_norm_krp(tt.context().get(), tt.get(), width, seed, static_cast<int>(rng), &v));
    return v;
}

inline double norm_exact(const TTTensor& tt) {
    double v = 0.0;
    check(ttr_norm_exact(tt.context().get(), tt.get(), &v));
    return v;
}

inline double relative_error(const TTTensor& a, const TTTensor& b) {
    double v = 0.0;
    check(ttr_relative_error(a.context().get(), a.get(), b.get(), &v));
    return v;
}

inline TTTensor formal_sum(const std::vector<TTTensor>& terms) {
    if (terms.empty()) fail(Errc::EmptyTermList, "formal sum of no terms");
    std::vector<const ttr_tt*> hs;
    for (const auto& t : terms) hs.push_back(t.get());
    ttr_tt* out = nullptr;
    check(ttr_tt_formal_sum(terms.front().context().get(), hs.data(), static_cast<int>(hs.size()), &out));
    return TTTensor(out, terms.front().context());
}

inline TTTensor scaled(const TTTensor& tt, double alpha) {
    TTTensor out = formal_sum({tt});
    check(ttr_tt_scale(out.context().get(), out.get(), alpha));
    return out;
}

//! random_gaussian_tt (tensor.hpp:111): the reference's xoshiro stream, bitwise.
inline TTTensor random_gaussian_tt(const std::vector<Index>& mode_sizes, const std::vector<Index>& ranks,
                                   std::uint64_t seed, Context& ctx = Context::thread_default()) {
    if (ranks.size() != mode_sizes.size() + 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
    ttr_tt* out = nullptr;
    check(ttr_tt_random_gaussian(ctx.get(), static_cast<int64_t>(mode_sizes.size()), mode_sizes.data(), ranks.data(),
                                 seed, &out));
    return TTTensor(out, ctx);
}

//! dot (tensor.hpp:119): <a, b> by the core-contraction sweep.
inline double dot(const TTTensor& a, const TTTensor& b) {
    double v = 0.0;
    check(ttr_dot(a.context().get(), a.get(), b.get(), &v));
    return v;
}

//! GaussianStream (rng.hpp:12-35). Xoshiro: the reference's sequential stream;
//! Philox: the device generator, whose state is the next global KRP column.
class GaussianStream {
public:
    explicit GaussianStream(std::uint64_t seed, RngMode rng = RngMode::Xoshiro) {
        ttr_stream* s = nullptr;
        check(ttr_stream_create(seed, static_cast<int>(rng), &s));
        h_.reset(s, &ttr_stream_destroy);
    }
    ttr_stream* get() const { return h_.get(); }

private:
    std::shared_ptr<ttr_stream> h_;
};

//! GaussianFactorSet (sketch.hpp:13-22): Omega_start..Omega_d, device-resident.
class GaussianFactorSet {
public:
    GaussianFactorSet(ttr_factors* owned, Context& ctx) : h_(owned, &ttr_factors_destroy), ctx_(&ctx) {}
    Index start_mode() const { return shape()[0]; }
    Index cols() const { return shape()[2]; }
    Index num_modes() const { return shape()[1]; }
    //! Omega_k (n_k x cols) copied to the host.
    Matrix at_mode(Index k, Index n_k) const {
        Matrix m(n_k, cols());
        check(ttr_factors_download(ctx_->get(), h_.get(), k, m.data()));
        return m;
    }
    ttr_factors* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    std::vector<Index> shape() const {
        int64_t a = 0, b = 0, c = 0;
        check(ttr_factors_shape(h_.get(), &a, &b, &c));
        return {a, b, c};
    }
    std::shared_ptr<ttr_factors> h_;
    Context* ctx_;
};

inline GaussianFactorSet draw_gaussian_factors(const TTTensor& tt, Index start_mode, Index cols,
                                               GaussianStream& stream) {
    ttr_factors* out = nullptr;
    check(ttr_draw_gaussian_factors(tt.context().get(), tt.get(), start_mode, cols, stream.get(), &out));
    return GaussianFactorSet(out, tt.context());
}

inline void append_gaussian_columns(GaussianFactorSet& set, Index extra, GaussianStream& stream) {
    check(ttr_append_gaussian_columns(set.context().get(), set.get(), extra, stream.get()));
}

//! PartialContractionSet (sketch.hpp:35-44): W_start..W_d, device-resident.
class PartialContractionSet {
public:
    PartialContractionSet(ttr_contractions* owned, Context& ctx) : h_(owned, &ttr_contractions_destroy), ctx_(&ctx) {}
    Index start_mode() const {
        int64_t s = 0;
        check(ttr_contractions_shape(h_.get(), 0, &s, nullptr, nullptr, nullptr));
        return s;
    }
    //! W_k (r_{k-1} x cols_k) copied to the host.
    Matrix at_mode(Index k) const {
        int64_t rows = 0, cols = 0;
        check(ttr_contractions_shape(h_.get(), k, nullptr, nullptr, &rows, &cols));
        Matrix m(rows, cols);
        check(ttr_contractions_download(ctx_->get(), h_.get(), k, m.data()));
        return m;
    }
    ttr_contractions* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    std::shared_ptr<ttr_contractions> h_;
    Context* ctx_;
};

inline PartialContractionSet krp_partial_contractions_rl(const TTTensor& tt, const GaussianFactorSet& factors) {
    ttr_contractions* out = nullptr;
    check(ttr_krp_partial_contractions_rl(tt.context().get(), tt.get(), factors.get(), &out));
    return PartialContractionSet(out, tt.context());
}

inline void append_krp_contractions(PartialContractionSet& set, const TTTensor& tt, const GaussianFactorSet& fresh) {
    check(ttr_append_krp_contractions(tt.context().get(), set.get(), tt.get(), fresh.get()));
}

//! generate_residual_sketch (round_rand.hpp:37-39).
inline Matrix generate_residual_sketch(const TTTensor& tt, const Matrix& z, const Matrix& q, PartialContractionSet& w,
                                       Index k, Index b, GaussianStream& stream) {
    Matrix s(z.rows(), b > 0 ? b : 0);
    check(ttr_generate_residual_sketch(tt.context().get(), tt.get(), z.rows(), z.cols(), z.data(), q.cols(),
                                       q.cols() ? q.data() : nullptr, w.get(), k, b, stream.get(), s.data()));
    return s;
}

//! residual_norm_estimate (sketch.hpp:67): ||S||_F / sqrt(block).
inline double residual_norm_estimate(const Matrix& s, Index block, Context& ctx = Context::thread_default()) {
    double v = 0.0;
    check(ttr_residual_norm_estimate(ctx.get(), s.rows(), s.cols(), s.data(), block, &v));
    return v;
}

// ---- TT-GMRES cookie harness (solver.hpp) ----------------------------------

//! KroneckerSumOperator (solver.hpp:12-21): terms[i][k-1] = A_{i,k}; the
//! factors are uploaded once (the device operator is kept alongside).
struct KroneckerSumOperator {
    std::vector<std::vector<Matrix>> terms;
    std::shared_ptr<ttr_kron_op> dev;
    static KroneckerSumOperator of(std::vector<std::vector<Matrix>> terms, Context& ctx = Context::thread_default()) {
        if (terms.empty()) throw Error(Errc::InvalidArgument, "operator needs at least one term");
        const std::size_t d = terms.front().size();
        if (d == 0) throw Error(Errc::InvalidArgument, "operator term needs at least one factor");
        std::vector<int64_t> n;
        for (const auto& a : terms.front()) n.push_back(a.rows());
        std::vector<double> flat;
        for (const auto& term : terms) {
            if (term.size() != d) throw Error(Errc::ModeSizeMismatch, "operator terms have unequal order");
            for (std::size_t k = 0; k < d; ++k) {
                if (term[k].rows() != term[k].cols() || term[k].rows() != n[k])
                    throw Error(Errc::ModeSizeMismatch, "operator factors must be square and consistent");
                flat.insert(flat.end(), term[k].a.begin(), term[k].a.end());
            }
        }
        ttr_kron_op* h = nullptr;
        check(ttr_kron_op_create(ctx.get(), static_cast<int64_t>(terms.size()), static_cast<int64_t>(d), n.data(),
                                 flat.data(), &h));
        KroneckerSumOperator op;
        op.terms = std::move(terms);
        op.dev.reset(h, &ttr_kron_op_destroy);
        return op;
    }
    Index num_terms() const { return static_cast<Index>(terms.size()); }
    Index order() const { return static_cast<Index>(terms.front().size()); }
    std::vector<Index> mode_sizes() const {
        std::vector<Index> out;
        for (const auto& a : terms.front()) out.push_back(a.rows());
        return out;
    }
};

struct CookieProblem {
    KroneckerSumOperator op;
    TTTensor rhs;
};

//! build_cookie_problem (solver.hpp:32-40): assembled on the host and the
//! device by the same formulas (the host factors stay in op.terms).
inline CookieProblem build_cookie_problem(Index num_param_modes, Index grid_size, Index num_param_samples,
                                          double rho_min, double rho_max, Context& ctx = Context::thread_default()) {
    ttr_kron_op* h = nullptr;
    ttr_tt* rhs = nullptr;
    check(ttr_cookie_problem(ctx.get(), num_param_modes, grid_size, num_param_samples, rho_min, rho_max, &h, &rhs));
    std::shared_ptr<ttr_kron_op> dev(h, &ttr_kron_op_destroy);
    TTTensor b(rhs, ctx);
    // host copies of the factors (the reference keeps them in op.terms)
    int64_t nterms = 0, d = 0;
    check(ttr_kron_op_shape(h, &nterms, &d, nullptr));
    std::vector<int64_t> n(static_cast<std::size_t>(d));
    check(ttr_kron_op_shape(h, &nterms, &d, n.data()));
    std::size_t tot = 0;
    for (int64_t k : n) tot += static_cast<std::size_t>(k * k);
    std::vector<double> flat(tot * static_cast<std::size_t>(nterms));
    check(ttr_kron_op_factors(h, flat.data()));
    KroneckerSumOperator op;
    op.dev = dev;
    std::size_t off = 0;
    for (int64_t i = 0; i < nterms; ++i) {
        std::vector<Matrix> term;
        for (int64_t k : n) {
            Matrix a(k, k);
            std::copy(flat.begin() + static_cast<std::ptrdiff_t>(off), flat.begin() + static_cast<std::ptrdiff_t>(off + k * k),
                      a.a.begin());
            off += static_cast<std::size_t>(k * k);
            term.push_back(std::move(a));
        }
        op.terms.push_back(std::move(term));
    }
    return CookieProblem{std::move(op), std::move(b)};
}

//! apply_operator (solver.hpp:42-44): the s-term sum A x.
inline TTSum apply_operator(const KroneckerSumOperator& op, const TTTensor& x) {
    std::vector<ttr_tt*> outs(static_cast<std::size_t>(op.num_terms()), nullptr);
    check(ttr_apply_operator(x.context().get(), op.dev.get(), x.get(), outs.data()));
    std::vector<TTTensor> terms;
    for (ttr_tt* t : outs) terms.emplace_back(t, x.context());
    return TTSum::of(std::move(terms));
}

enum class RoundingStrategy { Deterministic = TTR_GMRES_DETERMINISTIC, RandOrthTT = TTR_GMRES_RAND_ORTH_TT,
                              AdaptiveKRPSum = TTR_GMRES_ADAPTIVE_KRP_SUM };

struct GMRESConfig {  // solver.hpp:48-64
    double rel_tolerance = 1e-8;
    Index max_iterations = 200;
    RoundingStrategy strategy = RoundingStrategy::Deterministic;
    double rounding_tolerance = 0.0;
    std::uint64_t seed = 0;
    bool track_true_residual = true;
    bool mean_field_preconditioner = true;
    RngMode rng = RngMode::Xoshiro;  //!< sketch generator of the randomized strategies
};

struct GMRESResult {  // solver.hpp:66-78
    TTTensor solution;
    std::vector<double> residual_history, true_residual_history;
    std::vector<Index> max_rank_history;
    std::vector<double> rounding_seconds_history;
    double rounding_seconds = 0.0;
    Index iterations = 0;
    bool converged = false;
};

//! tt_gmres (solver.hpp:80-82) on the device; throws Breakdown as the reference.
inline GMRESResult tt_gmres(const KroneckerSumOperator& op, const TTTensor& rhs, const GMRESConfig& cfg) {
    ttr_gmres_cfg c{cfg.rel_tolerance, cfg.max_iterations, static_cast<int>(cfg.strategy), cfg.rounding_tolerance,
                    cfg.seed, cfg.track_true_residual ? 1 : 0, cfg.mean_field_preconditioner ? 1 : 0,
                    static_cast<int>(cfg.rng)};
    const std::size_t m = static_cast<std::size_t>(cfg.max_iterations > 0 ? cfg.max_iterations : 1);
    std::vector<double> rh(m), th(m), sh(m);
    std::vector<int64_t> kh(m);
    ttr_gmres_result r{0, 0, 0.0, rh.data(), th.data(), kh.data(), sh.data()};
    ttr_tt* sol = nullptr;
    check(ttr_tt_gmres(rhs.context().get(), op.dev.get(), rhs.get(), &c, &r, &sol));
    const std::size_t n = static_cast<std::size_t>(r.iterations);
    GMRESResult out{TTTensor(sol, rhs.context()), {}, {}, {}, {}, r.rounding_seconds, r.iterations, r.converged != 0};
    out.residual_history.assign(rh.begin(), rh.begin() + n);
    if (cfg.track_true_residual) out.true_residual_history.assign(th.begin(), th.begin() + n);
    out.max_rank_history.assign(kh.begin(), kh.begin() + n);
    out.rounding_seconds_history.assign(sh.begin(), sh.begin() + n);
    return out;
}

namespace flops {
struct Counts {  // flops.hpp:12-20
    std::uint64_t gemm = 0, qr = 0, svd = 0, sketch = 0, rng = 0;
    std::uint64_t total() const noexcept { return gemm + qr + svd; }
};
inline Counts counters(Context& ctx = Context::thread_default()) {
    ttr_counts c{};
    check(ttr_counters(ctx.get(), &c));
    return Counts{c.gemm, c.qr, c.svd, c.sketch, c.rng};
}
inline void reset(Context& ctx = Context::thread_default()) { check(ttr_counters_reset(ctx.get())); }
}  // namespace flops

}  // namespace ttround
