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
//   round_deterministic (tolerance / ranks) orthogonalize.hpp:50,54
//   estimate_norm_krp                       sketch.hpp:63
//   norm_exact / relative_error / formal_sum / scaled   tensor.hpp:172-191
//   flops::counters / reset                 flops.hpp:12-25
//
// Differences a caller sees: cores live in HBM (construct from host cores,
// read back with cores()); every call takes an optional Context (default: a
// per-thread context on device 0); the sketch generator defaults to the
// counter-based Philox stream (RngMode::Xoshiro reproduces the reference's
// sequential stream). Errors are rethrown as ttround::Error with the same
// Errc kinds the reference uses.
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

[[noreturn]] inline void fail(Errc code, const std::string& what) { throw Error(code, what); }

inline void check(ttr_status s) {
    if (s == TTR_OK) return;
    const std::string msg = ttr_last_error();
    if (s >= 1 && s <= 15) throw Error(static_cast<Errc>(s - 1), msg, s);
    throw Error(Errc::InvalidArgument, "device failure: " + msg, s);  // CUDA / OOM / no device
}

enum class RngMode : int { Xoshiro = TTR_RNG_XOSHIRO, Philox = TTR_RNG_PHILOX };

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
    RngMode rng = RngMode::Philox;
};

inline TTTensor round_fixed_krp(const TTTensor& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                                RngMode rng = RngMode::Philox) {
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
                                   RngMode rng = RngMode::Philox) {
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
                                       RngMode rng = RngMode::Philox) {
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

inline double estimate_norm_krp(const TTTensor& tt, Index width, std::uint64_t seed, RngMode rng = RngMode::Philox) {
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
