// sketch_api.cu — the reference's sketch-level API and the remaining tensor
// entry points at the C boundary, over device-resident objects:
//
//   ttr_stream        GaussianStream               rng.hpp:12-35
//   ttr_factors       GaussianFactorSet            sketch.hpp:13-22
//     ttr_draw_gaussian_factors                    sketch.hpp:25-26, sketch.cpp:44-56
//     ttr_append_gaussian_columns                  sketch.hpp:29, sketch.cpp:58-65
//   ttr_contractions  PartialContractionSet        sketch.hpp:35-44
//     ttr_krp_partial_contractions_rl              sketch.hpp:47-48, sketch.cpp:67-78
//     ttr_append_krp_contractions                  sketch.hpp:52-53, sketch.cpp:80-92
//   ttr_generate_residual_sketch                   round_rand.hpp:37-39, round_rand.cpp:80-94
//   ttr_residual_norm_estimate                     sketch.hpp:67, sketch.cpp:121-124
//   ttr_dot                                        tensor.hpp:119, tensor.cpp:244-256
//   ttr_tt_random_gaussian                         tensor.hpp:111, tensor.cpp:217-242
//   ttr_tt_upload_cores (TTTensor(vector<Core>))   tensor.hpp:63, tensor.cpp:66-79
//
// Every contraction runs through the same KRP step kernel as the rounding
// drivers (krp_step: TMA-fed DMMA GEMM over H(X_k) with the Omega*W scaling
// in the operand path), so a column's bits do not depend on how many columns
// are contracted together: appends equal one-shot contractions bitwise.
#include <cmath>
#include <cstring>

#include "capi_util.h"
#include "common.cuh"
#include "rng_host.h"
#include "tt_round.h"

using namespace ttr;
using namespace ttr::capi;

// GaussianStream: TTR_RNG_XOSHIRO is the reference's sequential stream (host
// state, bitwise rng.cpp:23-67); TTR_RNG_PHILOX is the counter-based device
// generator, whose state is the next global column index (a draw of c columns
// takes columns [next, next + c) of every mode's factor).
struct ttr_stream {
    std::uint64_t seed;
    int mode;
    XoshiroGauss xo;
    i64 next_col = 0;
    ttr_stream(std::uint64_t s, int m) : seed(s), mode(m), xo(s) {}
};

struct ttr_factors {
    Ctx* c;
    i64 start = 2, cols = 0, col0 = 0;  // Philox: columns [col0, col0 + cols)
    int mode = TTR_RNG_PHILOX;
    std::vector<i64> rows, ld;           // per mode start..d (index k - start)
    std::vector<DBuf> om;                // n_k x cols, leading dim ld (even)
};

struct ttr_contractions {
    Ctx* c;
    i64 start = 2;
    std::vector<i64> rows, cols, ld;  // W_k: r_{k-1} x cols[k - start], leading dim ld
    std::vector<DBuf> W;
};

namespace ttr {

void check_finite(Ctx& c, const TTDev& t) {
    std::vector<std::pair<const double*, std::size_t>> spans;
    for (i64 k = 0; k < t.d(); ++k) spans.emplace_back(t.core(k), static_cast<std::size_t>(t.core_size(k)));
    if (!all_finite(c, spans)) fail(Errc::InvalidArgument, "core entries must be finite");
}

double dot(Ctx& c, const TTDev& a, const TTDev& b) {
    if (a.n != b.n) fail(Errc::ModeSizeMismatch, "dot: mode sizes differ");
    DBuf w(c, 1);  // r_b(k) x r_a(k), starts as the 1 x 1 identity
    fill(c, w.p, 1, 1.0);
    for (i64 k = 0; k < a.d(); ++k) {
        const i64 ral = a.r[k], rar = a.r[k + 1], rbl = b.r[k], rbr = b.r[k + 1], n = a.n[k];
        DBuf hz(c, static_cast<std::size_t>(rbl * n * rar));  // w * H(A_k): r_b(k-1) x (n r_a(k))
        gemm(c, false, rbl, n * rar, ral, 1.0, w.p, rbl, a.core(k), ral, 0.0, hz.p, rbl);
        DBuf wn(c, static_cast<std::size_t>(rbr * rar));      // V(B_k)^T V(hz): r_b(k) x r_a(k)
        gemm(c, true, rbr, rar, rbl * n, 1.0, b.core(k), rbl * n, hz.p, rbl * n, 0.0, wn.p, rbr);
        w = std::move(wn);
    }
    TTR_CUDA(cudaMemcpyAsync(c.host_scalars, w.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    return c.host_scalars[0];
}

std::unique_ptr<TTDev> random_gaussian_tt(Ctx& c, const std::vector<i64>& n, const std::vector<i64>& r,
                                          std::uint64_t seed) {
    const i64 d = static_cast<i64>(n.size());
    if (d < 1 || static_cast<i64>(r.size()) != d + 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
    if (r.front() != 1 || r.back() != 1) fail(Errc::InvalidRankChain, "boundary ranks must be 1");
    for (i64 v : r)
        if (v < 1) fail(Errc::InvalidRankChain, "ranks must be positive");
    for (i64 v : n)
        if (v < 1) fail(Errc::InvalidRankChain, "mode sizes must be positive");
    auto t = std::make_unique<TTDev>(c, n, r);
    XoshiroGauss xo(seed);
    for (i64 k = 0; k < d; ++k) {
        const double sigma = 1.0 / std::sqrt(static_cast<double>(r[k]) * n[k] * r[k + 1]);
        std::vector<double> host(static_cast<std::size_t>(t->core_size(k)));
        for (auto& v : host) v = sigma * xo.next();
        TTR_CUDA(cudaMemcpyAsync(t->core(k), host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice,
                                 c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));  // host staging lifetime
    }
    return t;
}

}  // namespace ttr

namespace {

// Omega columns [dst_col, dst_col + cols) of every factor of f, drawn from the stream.
void draw_into(Ctx& c, ttr_factors& f, i64 dst_col, i64 cols, ttr_stream& s, i64 philox_col0) {
    for (std::size_t q = 0; q < f.om.size(); ++q) {
        const i64 k = f.start + static_cast<i64>(q), nk = f.rows[q];
        double* dst = f.om[q].p + dst_col * f.ld[q];
        if (s.mode == TTR_RNG_PHILOX) {
            philox_factor(c, s.seed, k, nk, cols, philox_col0, dst, f.ld[q]);
        } else {
            auto host = s.xo.matrix(nk, cols);  // rng.cpp:62-67, column-major
            TTR_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * f.ld[q], host.data(), sizeof(double) * nk,
                                       sizeof(double) * nk, cols, cudaMemcpyHostToDevice, c.stream));
            TTR_CUDA(cudaStreamSynchronize(c.stream));
        }
        c.counts.rng += static_cast<std::uint64_t>(nk * cols);
    }
}

// contract_tail (sketch.cpp:29-40) of tt against the factors of f: W_k for
// k = f.start..d (r_{k-1} x f.cols each, leading dim even_ld(r_{k-1})).
std::vector<DBuf> contract(Ctx& c, const TTDev& t, const ttr_factors& f, std::vector<i64>& ldw) {
    const i64 d = t.d(), cols = f.cols;
    if (f.start < 2) fail(Errc::InvalidArgument, "contraction start mode must be >= 2");
    if (f.start + static_cast<i64>(f.om.size()) - 1 != d)
        fail(Errc::ModeSizeMismatch, "factor set must cover modes start..d of the tensor");
    for (i64 k = f.start; k <= d; ++k)
        if (f.rows[static_cast<std::size_t>(k - f.start)] != t.n[k - 1])
            fail(Errc::ModeSizeMismatch, "factor rows must match the mode size");
    const i64 ldwt = even_ld(cols);
    std::vector<DBuf> W, Wt(static_cast<std::size_t>(d + 2));
    ldw.clear();
    for (i64 k = f.start; k <= d; ++k) {
        ldw.push_back(even_ld(t.r[k - 1]));
        W.emplace_back(c, static_cast<std::size_t>(ldw.back() * cols));
        if (k > f.start) Wt[k] = DBuf(c, static_cast<std::size_t>(ldwt * t.r[k - 1]));
    }
    DBuf ones(c, static_cast<std::size_t>(ldwt));
    fill(c, ones.p, static_cast<std::size_t>(ldwt), 1.0);
    SketchScope scope(c);
    for (i64 k = d; k >= f.start; --k) {
        const std::size_t q = static_cast<std::size_t>(k - f.start);
        krp_step(c, t.r[k - 1], t.n[k - 1], t.r[k], cols, t.core(k - 1), f.om[q].p, f.ld[q],
                 k == d ? ones.p : Wt[k + 1].p, ldwt, W[q].p, ldw[q], k > f.start ? Wt[k].p : nullptr, ldwt,
                 k == d);
    }
    return W;
}

void check_ctx(ttr_ctx* ctx, const Ctx* owner) {
    need(ctx != nullptr && owner == &ctx->c, "object belongs to another context");
}

std::unique_ptr<ttr_factors> draw_factors(Ctx& c, const TTDev& t, i64 start_mode, i64 cols, ttr_stream& stream) {
    const i64 d = t.d();
    if (start_mode < 2 || start_mode > d) fail(Errc::InvalidArgument, "factor start mode must lie in [2, d]");
    if (cols < 1) fail(Errc::InvalidArgument, "factor column count must be >= 1");
    auto f = std::make_unique<ttr_factors>();
    f->c = &c;
    f->start = start_mode;
    f->cols = cols;
    f->mode = stream.mode;
    f->col0 = stream.next_col;
    for (i64 k = start_mode; k <= d; ++k) {
        f->rows.push_back(t.n[k - 1]);
        f->ld.push_back(even_ld(t.n[k - 1]));
        f->om.emplace_back(c, static_cast<std::size_t>(f->ld.back() * cols));
    }
    draw_into(c, *f, 0, cols, stream, f->col0);
    if (stream.mode == TTR_RNG_PHILOX) stream.next_col += cols;
    return f;
}

void append_contractions(Ctx& c, ttr_contractions& w, const TTDev& t, const ttr_factors& fresh) {
    if (fresh.start < w.start) fail(Errc::InvalidArgument, "append must not precede the contraction start mode");
    if (w.start + static_cast<i64>(w.W.size()) - 1 != t.d())
        fail(Errc::ModeSizeMismatch, "contraction set does not match the tensor order");
    std::vector<i64> ldf;
    auto add = contract(c, t, fresh, ldf);
    for (i64 k = fresh.start; k <= t.d(); ++k) {
        const std::size_t q = static_cast<std::size_t>(k - w.start), a = static_cast<std::size_t>(k - fresh.start);
        if (w.rows[q] != t.r[k - 1]) fail(Errc::ModeSizeMismatch, "contraction rows must match the ranks");
        const i64 grown_cols = w.cols[q] + fresh.cols;
        DBuf grown(c, static_cast<std::size_t>(w.ld[q] * grown_cols));
        TTR_CUDA(cudaMemcpyAsync(grown.p, w.W[q].p, sizeof(double) * w.ld[q] * w.cols[q], cudaMemcpyDeviceToDevice,
                                 c.stream));
        TTR_CUDA(cudaMemcpy2DAsync(grown.p + w.ld[q] * w.cols[q], sizeof(double) * w.ld[q], add[a].p,
                                   sizeof(double) * ldf[a], sizeof(double) * w.rows[q], fresh.cols,
                                   cudaMemcpyDeviceToDevice, c.stream));
        w.W[q] = std::move(grown);
        w.cols[q] = grown_cols;
    }
}

}  // namespace

extern "C" {

ttr_status ttr_stream_create(uint64_t seed, int rng_mode, ttr_stream** out) {
    return guard([&] {
        need(out != nullptr, "null argument");
        need(rng_mode == TTR_RNG_PHILOX || rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
        *out = new ttr_stream(seed, rng_mode);
    });
}

ttr_status ttr_stream_destroy(ttr_stream* s) {
    delete s;
    return TTR_OK;
}

ttr_status ttr_draw_gaussian_factors(ttr_ctx* ctx, const ttr_tt* tt, int64_t start_mode, int64_t cols,
                                     ttr_stream* stream, ttr_factors** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(stream && out, "null argument");
        *out = draw_factors(ctx->c, *tt->t, start_mode, cols, *stream).release();
    });
}

ttr_status ttr_append_gaussian_columns(ttr_ctx* ctx, ttr_factors* f, int64_t extra, ttr_stream* stream) {
    return guard_ctx(ctx, [&] {
        need(f && stream, "null argument");
        check_ctx(ctx, f->c);
        if (extra < 1) fail(Errc::InvalidArgument, "factor column count must be >= 1");
        if (stream->mode != f->mode) fail(Errc::InvalidArgument, "stream and factor set use different generators");
        Ctx& c = ctx->c;
        for (std::size_t q = 0; q < f->om.size(); ++q) {
            DBuf grown(c, static_cast<std::size_t>(f->ld[q] * (f->cols + extra)));
            TTR_CUDA(cudaMemcpyAsync(grown.p, f->om[q].p, sizeof(double) * f->ld[q] * f->cols,
                                     cudaMemcpyDeviceToDevice, c.stream));
            f->om[q] = std::move(grown);
        }
        // Philox: the set's columns stay contiguous in the global column index
        draw_into(c, *f, f->cols, extra, *stream, f->col0 + f->cols);
        f->cols += extra;
        if (stream->mode == TTR_RNG_PHILOX) stream->next_col = std::max(stream->next_col, f->col0 + f->cols);
    });
}

ttr_status ttr_factors_upload(ttr_ctx* ctx, int64_t start_mode, int64_t nmodes, const int64_t* rows, int64_t cols,
                              const double* host, ttr_factors** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && rows && host && out, "null argument");
        if (start_mode < 2) fail(Errc::InvalidArgument, "factor start mode must lie in [2, d]");
        if (cols < 1 || nmodes < 1) fail(Errc::InvalidArgument, "factor column count must be >= 1");
        auto f = std::make_unique<ttr_factors>();
        f->c = &ctx->c;
        f->start = start_mode;
        f->cols = cols;
        i64 off = 0;
        for (i64 q = 0; q < nmodes; ++q) {
            need(rows[q] >= 1, "factor rows must be positive");
            f->rows.push_back(rows[q]);
            f->ld.push_back(even_ld(rows[q]));
            f->om.emplace_back(ctx->c, static_cast<std::size_t>(f->ld.back() * cols));
            TTR_CUDA(cudaMemcpy2DAsync(f->om.back().p, sizeof(double) * f->ld.back(), host + off,
                                       sizeof(double) * rows[q], sizeof(double) * rows[q], cols,
                                       cudaMemcpyHostToDevice, ctx->c.stream));
            off += rows[q] * cols;
        }
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
        *out = f.release();
    });
}

ttr_status ttr_factors_shape(const ttr_factors* f, int64_t* start_mode, int64_t* nmodes, int64_t* cols) {
    return guard([&] {
        need(f != nullptr, "null argument");
        if (start_mode) *start_mode = f->start;
        if (nmodes) *nmodes = static_cast<int64_t>(f->om.size());
        if (cols) *cols = f->cols;
    });
}

ttr_status ttr_factors_download(ttr_ctx* ctx, const ttr_factors* f, int64_t mode, double* host) {
    return guard_ctx(ctx, [&] {
        need(f && host, "null argument");
        check_ctx(ctx, f->c);
        const i64 q = mode - f->start;
        if (q < 0 || q >= static_cast<i64>(f->om.size())) fail(Errc::IndexOutOfRange, "mode outside the factor set");
        TTR_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * f->rows[q], f->om[q].p, sizeof(double) * f->ld[q],
                                   sizeof(double) * f->rows[q], f->cols, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_factors_destroy(ttr_factors* f) {
    delete f;
    return TTR_OK;
}

ttr_status ttr_krp_partial_contractions_rl(ttr_ctx* ctx, const ttr_tt* tt, const ttr_factors* f,
                                           ttr_contractions** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(f && out, "null argument");
        check_ctx(ctx, f->c);
        auto w = std::make_unique<ttr_contractions>();
        w->c = &ctx->c;
        w->start = f->start;
        w->W = contract(ctx->c, *tt->t, *f, w->ld);
        for (i64 k = f->start; k <= tt->t->d(); ++k) {
            w->rows.push_back(tt->t->r[k - 1]);
            w->cols.push_back(f->cols);
        }
        *out = w.release();
    });
}

ttr_status ttr_append_krp_contractions(ttr_ctx* ctx, ttr_contractions* w, const ttr_tt* tt, const ttr_factors* fresh) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(w && fresh, "null argument");
        check_ctx(ctx, w->c);
        check_ctx(ctx, fresh->c);
        append_contractions(ctx->c, *w, *tt->t, *fresh);
    });
}

ttr_status ttr_contractions_shape(const ttr_contractions* w, int64_t mode, int64_t* start_mode, int64_t* nmodes,
                                  int64_t* rows, int64_t* cols) {
    return guard([&] {
        need(w != nullptr, "null argument");
        if (start_mode) *start_mode = w->start;
        if (nmodes) *nmodes = static_cast<int64_t>(w->W.size());
        const i64 q = mode - w->start;
        if (rows || cols) {
            if (q < 0 || q >= static_cast<i64>(w->W.size())) fail(Errc::IndexOutOfRange, "mode outside the set");
            if (rows) *rows = w->rows[q];
            if (cols) *cols = w->cols[q];
        }
    });
}

ttr_status ttr_contractions_download(ttr_ctx* ctx, const ttr_contractions* w, int64_t mode, double* host) {
    return guard_ctx(ctx, [&] {
        need(w && host, "null argument");
        check_ctx(ctx, w->c);
        const i64 q = mode - w->start;
        if (q < 0 || q >= static_cast<i64>(w->W.size())) fail(Errc::IndexOutOfRange, "mode outside the set");
        TTR_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * w->rows[q], w->W[q].p, sizeof(double) * w->ld[q],
                                   sizeof(double) * w->rows[q], w->cols[q], cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_contractions_destroy(ttr_contractions* w) {
    delete w;
    return TTR_OK;
}

ttr_status ttr_generate_residual_sketch(ttr_ctx* ctx, const ttr_tt* tt, int64_t rows, int64_t z_cols,
                                        const double* host_z, int64_t q_cols, const double* host_q,
                                        ttr_contractions* w, int64_t k, int64_t b, ttr_stream* stream,
                                        double* host_s) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(w && stream && host_z && host_s && (q_cols == 0 || host_q), "null argument");
        check_ctx(ctx, w->c);
        const TTDev& t = *tt->t;
        if (b < 1) fail(Errc::InvalidArgument, "sketch block size must be >= 1");
        if (k < 1 || k >= t.d()) fail(Errc::InvalidArgument, "core index out of range");
        if (k + 1 < w->start || k + 1 > w->start + static_cast<i64>(w->W.size()) - 1)
            fail(Errc::InvalidArgument, "contraction set lacks mode k+1");
        need(rows >= 1 && q_cols >= 0, "bad matrix shape");
        const std::size_t q1 = static_cast<std::size_t>(k + 1 - w->start);
        if (z_cols != w->rows[q1]) fail(Errc::InvalidArgument, "z must have r_k columns");
        Ctx& c = ctx->c;
        const i64 used = q_cols, have = w->cols[q1];
        if (have < used + b) {  // round_rand.cpp:87-90: fresh factors for modes k+1..d, appended
            auto fresh = draw_factors(c, t, k + 1, used + b - have, *stream);
            append_contractions(c, *w, t, *fresh);
        }
        DBuf Z(c, static_cast<std::size_t>(rows * z_cols)), S(c, static_cast<std::size_t>(rows * b));
        TTR_CUDA(cudaMemcpyAsync(Z.p, host_z, sizeof(double) * rows * z_cols, cudaMemcpyHostToDevice, c.stream));
        gemm(c, false, rows, b, z_cols, 1.0, Z.p, rows, w->W[q1].p + used * w->ld[q1], w->ld[q1], 0.0, S.p, rows);
        if (used > 0) {  // S -= Q (Q^T S)
            DBuf Q(c, static_cast<std::size_t>(rows * used)), T(c, static_cast<std::size_t>(used * b));
            TTR_CUDA(cudaMemcpyAsync(Q.p, host_q, sizeof(double) * rows * used, cudaMemcpyHostToDevice, c.stream));
            gemm(c, true, used, b, rows, 1.0, Q.p, rows, S.p, rows, 0.0, T.p, used);
            gemm(c, false, rows, b, used, -1.0, Q.p, rows, T.p, used, 1.0, S.p, rows);
            TTR_CUDA(cudaMemcpyAsync(host_s, S.p, sizeof(double) * rows * b, cudaMemcpyDeviceToHost, c.stream));
            TTR_CUDA(cudaStreamSynchronize(c.stream));
        } else {
            TTR_CUDA(cudaMemcpyAsync(host_s, S.p, sizeof(double) * rows * b, cudaMemcpyDeviceToHost, c.stream));
            TTR_CUDA(cudaStreamSynchronize(c.stream));
        }
    });
}

ttr_status ttr_residual_norm_estimate(ttr_ctx* ctx, int64_t rows, int64_t cols, const double* host_s, int64_t block,
                                      double* out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out && (rows * cols == 0 || host_s), "null argument");
        if (block < 1) fail(Errc::InvalidArgument, "block size must be >= 1");
        need(rows >= 0 && cols >= 0, "bad matrix shape");
        double nrm = 0.0;
        if (rows * cols > 0) {
            Ctx& c = ctx->c;
            DBuf S(c, static_cast<std::size_t>(rows * cols));
            TTR_CUDA(cudaMemcpyAsync(S.p, host_s, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, c.stream));
            nrm = frob_norm(c, rows, cols, S.p, rows);
        }
        *out = nrm / std::sqrt(static_cast<double>(block));
    });
}

ttr_status ttr_dot(ttr_ctx* ctx, const ttr_tt* a, const ttr_tt* b, double* out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, a);
        check_same_ctx(ctx, b);
        need(out != nullptr, "null argument");
        *out = dot(ctx->c, *a->t, *b->t);
    });
}

ttr_status ttr_tt_random_gaussian(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r, uint64_t seed,
                                  ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        if (d < 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
        need(n && r, "null argument");
        *out = wrap(random_gaussian_tt(ctx->c, vec(n, d), vec(r, d + 1), seed));
    });
}

ttr_status ttr_tt_upload_cores(ttr_ctx* ctx, int64_t d, const int64_t* r_left, const int64_t* n,
                               const int64_t* r_right, const double* const* host_cores, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
        need(r_left && n && r_right && host_cores, "null argument");
        for (i64 k = 0; k < d; ++k)  // Core constructor (tensor.cpp:20-30)
            if (r_left[k] < 1 || n[k] < 1 || r_right[k] < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
        if (r_left[0] != 1 || r_right[d - 1] != 1) fail(Errc::BoundaryRankNotOne, "boundary TT ranks must be 1");
        for (i64 k = 0; k + 1 < d; ++k)
            if (r_right[k] != r_left[k + 1])
                fail(Errc::RankChainMismatch, "adjacent core ranks differ at position " + std::to_string(k + 1));
        std::vector<i64> nn(n, n + d), rr(static_cast<std::size_t>(d + 1));
        rr[0] = 1;
        for (i64 k = 0; k < d; ++k) rr[k + 1] = r_right[k];
        auto t = std::make_unique<TTDev>(ctx->c, nn, rr);
        for (i64 k = 0; k < d; ++k) {
            need(host_cores[k] != nullptr, "null core");
            TTR_CUDA(cudaMemcpyAsync(t->core(k), host_cores[k], sizeof(double) * t->core_size(k),
                                     cudaMemcpyHostToDevice, ctx->c.stream));
        }
        check_finite(ctx->c, *t);  // synchronises
        *out = wrap(std::move(t));
    });
}

}  // extern "C"
