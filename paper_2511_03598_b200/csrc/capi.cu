// capi.cu — the extern "C" boundary (include/ttround_b200.h). Catches every
// C++ exception and maps it to a ttr_status; messages are kept per thread.
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "tt_round.h"
#include "tt_gmres.h"
#include "capi_util.h"

using namespace ttr;
using namespace ttr::capi;

thread_local std::string g_last_error;  // declared in capi_util.h

extern "C" {

const char* ttr_last_error(void) { return g_last_error.c_str(); }
const char* ttr_version(void) { return "ttround_b200 0.1 (sm_100a, fp64 DMMA)"; }

ttr_status ttr_ctx_create(int device, void* stream, ttr_ctx** out) {
    return guard([&] {
        need(out != nullptr, "out is null");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw Error(TTR_ERR_NO_DEVICE, "no CUDA device available");
        need(device >= 0 && device < count, "device index out of range");
        TTR_CUDA(cudaSetDevice(device));
        auto* ctx = new ttr_ctx;
        ctx->c.device = device;
        TTR_CUDA(cudaDeviceGetAttribute(&ctx->c.sm_count, cudaDevAttrMultiProcessorCount, device));
        if (stream) {
            ctx->c.stream = static_cast<cudaStream_t>(stream);
        } else {
            TTR_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
            ctx->c.own_stream = true;
        }
        TTR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->c.host_scalars), 64 * sizeof(double)));
        // keep freed blocks in the stream-ordered pool (no release to the OS between calls)
        cudaMemPool_t pool;
        TTR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        std::uint64_t threshold = UINT64_MAX;
        TTR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        *out = ctx;
    });
}

ttr_status ttr_ctx_destroy(ttr_ctx* ctx) {
    return guard_ctx(ctx, [&] {
        if (!ctx) return;
        cudaSetDevice(ctx->c.device);
        if (ctx->c.work) cudaFreeAsync(ctx->c.work, ctx->c.stream);
        ctx->c.release_retired();
        cudaStreamSynchronize(ctx->c.stream);
        ctx->c.destroy_side();
        if (ctx->c.qr_xchg) cudaFree(ctx->c.qr_xchg);
        if (ctx->c.qr_flag) cudaFree(ctx->c.qr_flag);
        if (ctx->c.host_scalars) cudaFreeHost(ctx->c.host_scalars);
        if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
        delete ctx;
    });
}

ttr_status ttr_ctx_set_stream(ttr_ctx* ctx, void* stream) {
    return guard_ctx(ctx, [&] {
        need(ctx != nullptr, "null context");
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
        if (ctx->c.own_stream) {
            TTR_CUDA(cudaStreamDestroy(ctx->c.stream));
            ctx->c.own_stream = false;
        }
        if (stream) {
            ctx->c.stream = static_cast<cudaStream_t>(stream);
        } else {
            TTR_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
            ctx->c.own_stream = true;
        }
    });
}

ttr_status ttr_ctx_synchronize(ttr_ctx* ctx) {
    return guard_ctx(ctx, [&] {
        need(ctx != nullptr, "null context");
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_ctx_kernel_launches(ttr_ctx* ctx, uint64_t* out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        *out = ctx->c.launches;
    });
}

ttr_status ttr_tt_upload(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r, const double* host, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
        need(n && r && host, "null argument");
        auto t = std::make_unique<TTDev>(ctx->c, vec(n, d), vec(r, d + 1));
        t->upload(host);
        check_finite(ctx->c, *t);  // TTTensor ctor scan (tensor.cpp:75-78); synchronises
        *out = wrap(std::move(t));
    });
}

ttr_status ttr_tt_from_device(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r, const double* dev, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out && n && r && dev, "null argument");
        if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
        auto t = std::make_unique<TTDev>(ctx->c, vec(n, d), vec(r, d + 1));
        i64 o = 0;
        for (i64 k = 0; k < d; ++k) {
            TTR_CUDA(cudaMemcpyAsync(t->core(k), dev + o, sizeof(double) * t->core_size(k), cudaMemcpyDeviceToDevice,
                                     ctx->c.stream));
            o += t->core_size(k);
        }
        check_finite(ctx->c, *t);
        *out = wrap(std::move(t));
    });
}

ttr_status ttr_tt_shape(const ttr_tt* tt, int64_t* d, int64_t* n, int64_t* r, int64_t* total) {
    return guard([&] {
        need(tt && tt->t, "null tensor");
        const TTDev& t = *tt->t;
        if (d) *d = t.d();
        if (n) for (i64 k = 0; k < t.d(); ++k) n[k] = t.n[k];
        if (r) for (i64 k = 0; k <= t.d(); ++k) r[k] = t.r[k];
        if (total) *total = t.total();
    });
}

ttr_status ttr_tt_download(ttr_ctx* ctx, const ttr_tt* tt, double* host) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(host != nullptr, "null output");
        tt->t->download(host);
    });
}

// ---- TTF1 files (io.cpp:27-76): "TTF1", u32 d, u32 n[d], u32 r[d+1], then the
// cores' fp64 data in the reference layout, little-endian. Read/written
// through a pinned staging buffer straight to/from the device tensor.
ttr_status ttr_tt_write_ttf1(ttr_ctx* ctx, const ttr_tt* tt, const char* path) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(path != nullptr, "null path");
        const TTDev& t = *tt->t;
        std::FILE* f = std::fopen(path, "wb");
        if (!f) fail(Errc::IoError, std::string("cannot open ") + path + " for writing");
        bool ok = std::fwrite("TTF1", 1, 4, f) == 4;
        auto u32 = [&](i64 v) {
            const std::uint32_t w = static_cast<std::uint32_t>(v);
            ok = ok && std::fwrite(&w, sizeof w, 1, f) == 1;
        };
        u32(t.d());
        for (i64 v : t.n) u32(v);
        for (i64 v : t.r) u32(v);
        std::vector<double> host(static_cast<std::size_t>(t.total()));
        t.download(host.data());
        ok = ok && std::fwrite(host.data(), sizeof(double), host.size(), f) == host.size();
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) fail(Errc::IoError, std::string("failed writing ") + path);
    });
}

ttr_status ttr_tt_read_ttf1(ttr_ctx* ctx, const char* path, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && path && out, "null argument");
        std::FILE* f = std::fopen(path, "rb");
        if (!f) fail(Errc::IoError, std::string("cannot open ") + path);
        struct Closer {
            std::FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        char magic[4];
        if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "TTF1", 4) != 0)
            fail(Errc::IoError, std::string("not a TTF1 file: ") + path);
        auto u32 = [&]() {
            std::uint32_t w = 0;
            if (std::fread(&w, sizeof w, 1, f) != 1) fail(Errc::IoError, "unexpected end of TTF1 file");
            return static_cast<i64>(w);
        };
        const i64 d = u32();
        if (d == 0 || d > 64) fail(Errc::IoError, std::string("implausible TT order in ") + path);
        std::vector<i64> n(static_cast<std::size_t>(d)), r(static_cast<std::size_t>(d + 1));
        for (auto& v : n) v = u32();
        for (auto& v : r) v = u32();
        if (r.front() != 1 || r.back() != 1) fail(Errc::BoundaryRankNotOne, "TTF1 boundary ranks must be 1");
        i64 total = 0;
        for (i64 k = 0; k < d; ++k) {
            if (n[k] < 1 || r[k] < 1 || r[k + 1] < 1) fail(Errc::IoError, "invalid TTF1 dimensions");
            const i64 cnt = r[k] * n[k] * r[k + 1];
            if (cnt > (i64{1} << 34)) fail(Errc::IoError, std::string("implausible core size in ") + path);
            total += cnt;
        }
        auto t = std::make_unique<TTDev>(ctx->c, n, r);
        std::vector<double> host(static_cast<std::size_t>(total));
        if (std::fread(host.data(), sizeof(double), host.size(), f) != host.size())
            fail(Errc::IoError, "unexpected end of TTF1 file");
        t->upload(host.data());
        check_finite(ctx->c, *t);  // synchronises (host buffer lifetime); read_ttf1 builds a TTTensor
        *out = wrap(std::move(t));
    });
}

ttr_status ttr_tt_copy_from_host(ttr_ctx* ctx, ttr_tt* tt, const double* host) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(host != nullptr, "null input");
        tt->t->upload(host);
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_tt_download_core(ttr_ctx* ctx, const ttr_tt* tt, int64_t k, double* host) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(host != nullptr, "null argument");
        if (k < 0 || k >= tt->t->d()) fail(Errc::IndexOutOfRange, "core index out of range");
        TTR_CUDA(cudaMemcpyAsync(host, tt->t->core(k), sizeof(double) * tt->t->core_size(k), cudaMemcpyDeviceToHost,
                                 ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_tt_core_ptr(const ttr_tt* tt, int64_t k, const double** ptr) {
    return guard([&] {
        need(tt && tt->t && ptr, "null argument");
        if (k < 0 || k >= tt->t->d()) fail(Errc::IndexOutOfRange, "core index out of range");
        *ptr = tt->t->core(k);
    });
}

ttr_status ttr_tt_destroy(ttr_tt* tt) {
    return guard([&] { delete tt; });
}

ttr_status ttr_tt_random_philox(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r, uint64_t seed, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out && n && r, "null argument");
        if (d < 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
        *out = wrap(random_philox_tt(ctx->c, vec(n, d), vec(r, d + 1), seed));
    });
}

ttr_status ttr_tt_kernel_sum(ttr_ctx* ctx, int64_t d, int64_t n, int64_t r, int64_t terms, double ell, uint64_t seed,
                             ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        need(d >= 1 && n >= 1 && r >= 1 && terms >= 1 && ell > 0.0, "bad kernel-sum parameters");
        *out = wrap(kernel_sum_tt(ctx->c, d, n, r, terms, ell, seed));
    });
}

ttr_status ttr_tt_kernel_term(ttr_ctx* ctx, int64_t d, int64_t n, int64_t r, int64_t term, double ell, uint64_t seed,
                             ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        need(d >= 1 && n >= 1 && r >= 1 && term >= 0 && ell > 0.0, "bad kernel-sum parameters");
        *out = wrap(kernel_term_tt(ctx->c, d, n, r, term, ell, seed));
    });
}

ttr_status ttr_tt_formal_sum(ttr_ctx* ctx, const ttr_tt* const* terms, int count, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        std::vector<const TTDev*> ts;
        for (int i = 0; i < count; ++i) {
            check_same_ctx(ctx, terms[i]);
            ts.push_back(terms[i]->t.get());
        }
        *out = wrap(formal_sum(ctx->c, ts));
    });
}

ttr_status ttr_tt_scale(ttr_ctx* ctx, ttr_tt* tt, double alpha) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        scale_tt(ctx->c, *tt->t, alpha);
    });
}

ttr_status ttr_norm_exact(ttr_ctx* ctx, const ttr_tt* tt, double* out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        *out = norm_exact(ctx->c, *tt->t);
    });
}

ttr_status ttr_relative_error(ttr_ctx* ctx, const ttr_tt* a, const ttr_tt* b, double* out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, a);
        check_same_ctx(ctx, b);
        need(out != nullptr, "null output");
        if (a->t->n != b->t->n) fail(Errc::ModeSizeMismatch, "formal sum mode sizes differ");
        *out = relative_error(ctx->c, *a->t, *b->t);
    });
}

ttr_status ttr_round_fixed_krp(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* ranks, int64_t count, uint64_t seed,
                               int rng_mode, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        need(rng_mode == TTR_RNG_PHILOX || rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        *out = wrap(round_fixed_krp(ctx->c, *tt->t, vec(ranks, count), seed, rng_mode));
    });
}

ttr_status ttr_plan_fixed_krp(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* ranks, int64_t count, uint64_t seed,
                              int rng_mode, ttr_plan** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        auto* p = new ttr_plan;
        try {
            p->plan = std::make_unique<Plan>(ctx->c, *tt->t, vec(ranks, count), seed, rng_mode);
        } catch (...) {
            delete p;
            throw;
        }
        p->out.t = std::move(p->plan->out);
        p->ctx = ctx;
        *out = p;
    });
}

ttr_status ttr_plan_fixed_krp_host(ttr_ctx* ctx, ttr_tt* tt, const int64_t* ranks, int64_t count, uint64_t seed,
                                   const double* host_in, double* host_out, ttr_plan** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr && host_in != nullptr && host_out != nullptr, "null argument");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        auto* p = new ttr_plan;
        try {
            p->plan = std::make_unique<Plan>(ctx->c, *tt->t, vec(ranks, count), seed, TTR_RNG_PHILOX, host_in, host_out);
        } catch (...) {
            delete p;
            throw;
        }
        p->out.t = std::move(p->plan->out);
        p->ctx = ctx;
        *out = p;
    });
}

ttr_status ttr_plan_execute(ttr_plan* plan) {
    return guard([&] {
        need(plan && (plan->plan || plan->aplan), "null plan");
        if (plan->aplan) plan->aplan->execute();
        else plan->plan->execute();
    });
}

ttr_status ttr_plan_rerecords(const ttr_plan* plan, int64_t* count) {
    return guard([&] {
        need(plan && count, "null argument");
        *count = plan->aplan ? plan->aplan->rerecords : 0;
    });
}

ttr_status ttr_plan_output(ttr_plan* plan, const ttr_tt** out) {
    return guard([&] {
        need(plan && out, "null argument");
        *out = &plan->out;
    });
}

ttr_status ttr_plan_destroy(ttr_plan* plan) {
    return guard([&] {
        if (!plan) return;
        cudaStreamSynchronize(plan->ctx->c.stream);
        plan->aplan.reset();
        plan->plan.reset();
        delete plan;
    });
}

static AdaptiveCfg adaptive_cfg_of(const ttr_tt* tt, const ttr_adaptive_cfg* cfg) {
    need(cfg->rng_mode == TTR_RNG_PHILOX || cfg->rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
    AdaptiveCfg a;
    a.tolerance = cfg->tolerance;
    a.f_init = cfg->f_init;
    a.f_inc = cfg->f_inc;
    a.seed = cfg->seed;
    a.has_known_norm = cfg->has_known_norm != 0;
    a.known_norm = cfg->known_norm;
    if (cfg->max_rank_cap) {
        if (cfg->max_rank_cap_len != tt->t->d() - 1) fail(Errc::InvalidRanks, "max_rank_cap needs d-1 entries");
        for (int64_t k = 0; k < cfg->max_rank_cap_len; ++k)
            if (cfg->max_rank_cap[k] < 1) fail(Errc::InvalidRanks, "rank caps must be >= 1");
    }
    a.max_rank_cap = cfg->max_rank_cap;
    a.rng_mode = cfg->rng_mode;
    return a;
}

ttr_status ttr_plan_adaptive_krp(ttr_ctx* ctx, const ttr_tt* tt, const ttr_adaptive_cfg* cfg, ttr_plan** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(cfg && out, "null argument");
        AdaptiveCfg a = adaptive_cfg_of(tt, cfg);
        if (!(a.tolerance > 0.0 && a.tolerance < 1.0)) fail(Errc::InvalidArgument, "adaptive tolerance must lie in (0,1)");
        auto* p = new ttr_plan;
        try {
            p->aplan = std::make_unique<AdaptivePlan>(ctx->c, *tt->t, a, &p->out.t);
        } catch (...) {
            delete p;
            throw;
        }
        p->ctx = ctx;
        *out = p;
    });
}

ttr_status ttr_round_adaptive_krp(ttr_ctx* ctx, const ttr_tt* tt, const ttr_adaptive_cfg* cfg, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(cfg && out, "null argument");
        need(cfg->rng_mode == TTR_RNG_PHILOX || cfg->rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
        AdaptiveCfg a;
        a.tolerance = cfg->tolerance;
        a.f_init = cfg->f_init;
        a.f_inc = cfg->f_inc;
        a.seed = cfg->seed;
        a.has_known_norm = cfg->has_known_norm != 0;
        a.known_norm = cfg->known_norm;
        if (cfg->max_rank_cap) {
            if (cfg->max_rank_cap_len != tt->t->d() - 1) fail(Errc::InvalidRanks, "max_rank_cap needs d-1 entries");
            for (int64_t k = 0; k < cfg->max_rank_cap_len; ++k)
                if (cfg->max_rank_cap[k] < 1) fail(Errc::InvalidRanks, "rank caps must be >= 1");
        }
        a.max_rank_cap = cfg->max_rank_cap;
        a.rng_mode = cfg->rng_mode;
        *out = wrap(round_adaptive_krp(ctx->c, *tt->t, a, nullptr));
    });
}

ttr_status ttr_round_sum_adaptive_krp(ttr_ctx* ctx, const ttr_tt* const* terms, int64_t count, double eps, double f_inc,
                                      uint64_t seed, int rng_mode, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        if (count < 1 || !terms) fail(Errc::EmptyTermList, "sum of no TT terms");
        std::vector<const TTDev*> ts;
        for (int64_t i = 0; i < count; ++i) {
            check_same_ctx(ctx, terms[i]);
            ts.push_back(terms[i]->t.get());
        }
        need(rng_mode == TTR_RNG_PHILOX || rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
        *out = wrap(round_sum_adaptive_krp(ctx->c, ts, eps, f_inc, seed, rng_mode));
    });
}

ttr_status ttr_round_rand_orth_tt(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* ranks, int64_t count, uint64_t seed,
                                  int rng_mode, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        need(rng_mode == TTR_RNG_PHILOX || rng_mode == TTR_RNG_XOSHIRO, "unknown rng mode");
        *out = wrap(round_rand_orth_tt(ctx->c, *tt->t, vec(ranks, count), seed, rng_mode));
    });
}

ttr_status ttr_compression_pass(ttr_ctx* ctx, const ttr_tt* tt, double tau, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        *out = wrap(compression_pass(ctx->c, *tt->t, tau));
    });
}

ttr_status ttr_round_deterministic_tol(ttr_ctx* ctx, const ttr_tt* tt, double eps, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        *out = wrap(round_deterministic_tol(ctx->c, *tt->t, eps));
    });
}

ttr_status ttr_round_deterministic_ranks(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* ranks, int64_t count, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        *out = wrap(round_deterministic_ranks(ctx->c, *tt->t, vec(ranks, count)));
    });
}

ttr_status ttr_estimate_norm_krp(ttr_ctx* ctx, const ttr_tt* tt, int64_t width, uint64_t seed, int rng_mode, double* out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out != nullptr, "null output");
        *out = estimate_norm_krp(ctx->c, *tt->t, width, seed, rng_mode);
    });
}

ttr_status ttr_krp_partial_contractions(ttr_ctx* ctx, const ttr_tt* tt, int64_t start_mode, int64_t cols,
                                        const double* host_factors, uint64_t seed, int64_t col0, double* host_w) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(host_w != nullptr, "null output");
        krp_partial_contractions(ctx->c, *tt->t, start_mode, cols, host_factors, seed, col0, host_w);
    });
}

ttr_status ttr_philox_factor(ttr_ctx* ctx, uint64_t seed, int64_t mode, int64_t rows, int64_t cols, int64_t col0,
                             double* host_out) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_out, "null argument");
        need(rows >= 1 && cols >= 1, "empty shape");
        DBuf b(ctx->c, static_cast<std::size_t>(rows * cols));
        philox_factor(ctx->c, seed, mode, rows, cols, col0, b.p, rows);
        TTR_CUDA(cudaMemcpyAsync(host_out, b.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_thin_qr(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q, double* host_r) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_a, "null argument");
        need(m >= 1 && n >= 1, "empty shape");
        const i64 k = std::min(m, n);
        DBuf a(ctx->c, static_cast<std::size_t>(m * n)), q(ctx->c, static_cast<std::size_t>(m * k)),
            r(ctx->c, static_cast<std::size_t>(k * n));
        TTR_CUDA(cudaMemcpyAsync(a.p, host_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, ctx->c.stream));
        thin_qr(ctx->c, m, n, a.p, m, q.p, m, r.p, k);
        if (host_q) TTR_CUDA(cudaMemcpyAsync(host_q, q.p, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->c.stream));
        if (host_r) TTR_CUDA(cudaMemcpyAsync(host_r, r.p, sizeof(double) * k * n, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_thin_qr_speculative(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q,
                                   double* host_r, int* breakdown) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_a && breakdown, "null argument");
        need(m >= 1 && n >= 1, "empty shape");
        const i64 k = std::min(m, n);
        DBuf a(ctx->c, static_cast<std::size_t>(m * n)), q(ctx->c, static_cast<std::size_t>(m * k)),
            r(ctx->c, static_cast<std::size_t>(k * n));
        TTR_CUDA(cudaMemcpyAsync(a.p, host_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, ctx->c.stream));
        ctx->c.qr_flag_reset();
        ctx->c.qr_tag = 0;  // the blocked QR may take the Cholesky-QR panels (K4d/K4f)
        try {
            thin_qr(ctx->c, m, n, a.p, m, q.p, m, r.p, k);
        } catch (...) {
            ctx->c.qr_tag = -1;
            throw;
        }
        ctx->c.qr_tag = -1;
        if (host_q) TTR_CUDA(cudaMemcpyAsync(host_q, q.p, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->c.stream));
        if (host_r) TTR_CUDA(cudaMemcpyAsync(host_r, r.p, sizeof(double) * k * n, cudaMemcpyDeviceToHost, ctx->c.stream));
        *breakdown = ctx->c.qr_flag_read() >= 0 ? 1 : 0;
    });
}

ttr_status ttr_thin_qr_cholesky(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q,
                                double* host_r, int* breakdown) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_a && breakdown, "null argument");
        need(cholqr_fits(m, n), "shape outside the Cholesky-QR path (m >= n, n <= 416)");
        DBuf a(ctx->c, static_cast<std::size_t>(m * n)), q(ctx->c, static_cast<std::size_t>(m * n)),
            r(ctx->c, static_cast<std::size_t>(n * n));
        TTR_CUDA(cudaMemcpyAsync(a.p, host_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, ctx->c.stream));
        ctx->c.qr_flag_reset();
        thin_qr_cholesky(ctx->c, m, n, a.p, m, q.p, m, r.p, n);
        if (host_q) TTR_CUDA(cudaMemcpyAsync(host_q, q.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost, ctx->c.stream));
        if (host_r) TTR_CUDA(cudaMemcpyAsync(host_r, r.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost, ctx->c.stream));
        *breakdown = ctx->c.qr_flag_read() >= 0 ? 1 : 0;
    });
}

ttr_status ttr_dev_thin_qr_cholesky(ttr_ctx* ctx, int64_t m, int64_t n, const double* dA, int64_t lda, double* dQ,
                                    int64_t ldq, double* dR, int64_t ldr, int* breakdown) {
    return guard_ctx(ctx, [&] {
        need(ctx && dA && dQ && breakdown, "null argument");
        need(cholqr_fits(m, n) && lda >= m && ldq >= m && (!dR || ldr >= n), "bad shape");
        ctx->c.qr_flag_reset();
        thin_qr_cholesky(ctx->c, m, n, dA, lda, dQ, ldq, dR, ldr);
        *breakdown = ctx->c.qr_flag_read() >= 0 ? 1 : 0;
    });
}

ttr_status ttr_thin_qr_cholesky_batched(ttr_ctx* ctx, int64_t m, int64_t n, int64_t batch, const double* host_a,
                                        double* host_q, int* host_flags) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_a && host_q && host_flags && batch >= 0, "null argument");
        need(cholqr_small_fits(m, n), "shape outside the batched Cholesky-QR path (n <= 32, n <= m <= 2048)");
        if (batch == 0) return;
        const std::size_t tot = static_cast<std::size_t>(m * n * batch);
        DBuf a(ctx->c, tot), q(ctx->c, tot), f(ctx->c, static_cast<std::size_t>((batch + 1) / 2));
        int* flags = reinterpret_cast<int*>(f.p);
        TTR_CUDA(cudaMemcpyAsync(a.p, host_a, sizeof(double) * tot, cudaMemcpyHostToDevice, ctx->c.stream));
        TTR_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * batch, ctx->c.stream));
        cholqr_small_batched(ctx->c, m, n, a.p, m, m * n, q.p, m, m * n, batch, flags);
        TTR_CUDA(cudaMemcpyAsync(host_q, q.p, sizeof(double) * tot, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaMemcpyAsync(host_flags, flags, sizeof(int) * batch, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_dev_thin_qr_cholesky_batched(ttr_ctx* ctx, int64_t m, int64_t n, int64_t batch, const double* dA,
                                            int64_t lda, int64_t stride_a, double* dQ, int64_t ldq, int64_t stride_q,
                                            int* d_flags) {
    return guard_ctx(ctx, [&] {
        need(ctx && dA && dQ && d_flags && batch >= 0, "null argument");
        need(cholqr_small_fits(m, n) && lda >= m && ldq >= m && stride_a >= lda * n && stride_q >= ldq * n,
             "bad shape");
        if (batch > 0) cholqr_small_batched(ctx->c, m, n, dA, lda, stride_a, dQ, ldq, stride_q, batch, d_flags);
    });
}

ttr_status ttr_dev_thin_qr(ttr_ctx* ctx, int64_t m, int64_t n, const double* dA, int64_t lda, double* dQ, int64_t ldq,
                           double* dR, int64_t ldr) {
    return guard_ctx(ctx, [&] {
        need(ctx && dA, "null argument");
        need(m >= 1 && n >= 1 && lda >= m && (!dQ || ldq >= m), "bad shape");
        static const bool spec = std::getenv("TTR_QR_DEV_SPEC") != nullptr;  // tools/qr_bench.py: time the speculative panels
        ctx->c.qr_tag = spec ? 0 : -1;
        try {
            thin_qr(ctx->c, m, n, dA, lda, dQ, ldq, dR, ldr);
        } catch (...) {
            ctx->c.qr_tag = -1;
            throw;
        }
        ctx->c.qr_tag = -1;
    });
}

ttr_status ttr_dev_gemm(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, double alpha, const double* dA,
                        int64_t lda, const double* dB, int64_t ldb, double beta, double* dC, int64_t ldc) {
    return guard_ctx(ctx, [&] {
        need(ctx && dA && dB && dC, "null argument");
        gemm(ctx->c, trans_a != 0, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, ldc);
    });
}

ttr_status ttr_dev_gemm_batched(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                                const double* dA, int64_t lda, int64_t sA, const double* dB, int64_t ldb, int64_t sB,
                                double beta, double* dC, int64_t ldc, int64_t sC, int64_t batch) {
    return guard_ctx(ctx, [&] {
        need(ctx && dA && dB && dC, "null argument");
        need(batch >= 0, "negative batch");
        gemm_batched(ctx->c, trans_a != 0, m, n, k, alpha, dA, lda, sA, dB, ldb, sB, beta, dC, ldc, sC, batch);
    });
}

ttr_status ttr_gemm(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, const double* host_a, const double* host_b,
                    double* host_c) {
    return guard_ctx(ctx, [&] {
        need(ctx && host_a && host_b && host_c, "null argument");
        need(m >= 1 && n >= 1 && k >= 1, "empty shape");
        DBuf a(ctx->c, static_cast<std::size_t>(m * k)), b(ctx->c, static_cast<std::size_t>(k * n)),
            cc(ctx->c, static_cast<std::size_t>(m * n));
        TTR_CUDA(cudaMemcpyAsync(a.p, host_a, sizeof(double) * m * k, cudaMemcpyHostToDevice, ctx->c.stream));
        TTR_CUDA(cudaMemcpyAsync(b.p, host_b, sizeof(double) * k * n, cudaMemcpyHostToDevice, ctx->c.stream));
        gemm(ctx->c, trans_a != 0, m, n, k, 1.0, a.p, trans_a ? k : m, b.p, k, 0.0, cc.p, m);
        TTR_CUDA(cudaMemcpyAsync(host_c, cc.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost, ctx->c.stream));
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_ctx_enable_timing(ttr_ctx* ctx, int on) {
    return guard_ctx(ctx, [&] {
        need(ctx != nullptr, "null context");
        ctx->c.timing = on != 0;
    });
}

ttr_status ttr_ctx_phase_times(ttr_ctx* ctx, double* ms_out, uint64_t* count_out) {
    return guard_ctx(ctx, [&] {
        need(ctx != nullptr, "null context");
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
        for (int p = 0; p < kNumPhases; ++p) {
            double total = 0.0;
            for (auto& ev : ctx->c.phase_events[p]) {
                float ms = 0.f;
                TTR_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
                total += ms;
                cudaEventDestroy(ev.first);
                cudaEventDestroy(ev.second);
            }
            if (ms_out) ms_out[p] = total;
            if (count_out) count_out[p] = ctx->c.phase_events[p].size();
            ctx->c.phase_events[p].clear();
        }
    });
}

// ---- column-sharded sketch (multi-GPU config 5b) ----
ttr_status ttr_krp_sketch_into(ttr_ctx* ctx, const ttr_tt* tt, int64_t col0, int64_t ncols, uint64_t seed,
                               double* const* W_dev, const int64_t* ldw) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(W_dev && ldw, "null argument");
        const i64 d = tt->t->d();
        std::vector<double*> W(d + 2, nullptr);
        std::vector<i64> ld(d + 2, 0);
        for (i64 k = 2; k <= d; ++k) {
            W[k] = W_dev[k - 2];
            ld[k] = ldw[k - 2];
            need(W[k] && ld[k] >= tt->t->r[k - 1], "bad W buffer");
        }
        krp_sketch_into(ctx->c, *tt->t, col0, ncols, seed, W, ld);
    });
}

ttr_status ttr_round_fixed_krp_from_sketch(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* ranks, int64_t count,
                                           const double* const* W_dev, const int64_t* ldw, int64_t width, ttr_tt** out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(out && W_dev && ldw, "null argument");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        auto r = fixed_krp_ranks(*tt->t, vec(ranks, count));
        const i64 d = tt->t->d();
        for (i64 k = 1; k < d; ++k) need(r[k] <= width, "sketch narrower than the target ranks");
        std::vector<const double*> W(d + 2, nullptr);
        std::vector<i64> ld(d + 2, 0);
        for (i64 k = 2; k <= d; ++k) {
            W[k] = W_dev[k - 2];
            ld[k] = ldw[k - 2];
        }
        auto o = std::make_unique<TTDev>(ctx->c, tt->t->n, r);
        rand_orth_sweep(ctx->c, *tt->t, width, W, ld, *o);
        *out = wrap(std::move(o));
    });
}

// ---- batches of independent tensors (config 5a) ----
ttr_status ttr_batch_upload(ttr_ctx* ctx, int64_t batch, int64_t d, const int64_t* n, const int64_t* r,
                            const double* host, ttr_batch** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out && n && r && host, "null argument");
        if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
        auto t = std::make_unique<TTBatch>(ctx->c, batch, vec(n, d), vec(r, d + 1));
        const i64 tot = t->total();
        // padding between cores is zeroed so one scan covers the whole batch
        TTR_CUDA(cudaMemsetAsync(t->buf.p, 0, sizeof(double) * t->stride * batch, ctx->c.stream));
        for (i64 b = 0; b < batch; ++b) {
            i64 o = 0;
            for (i64 k = 0; k < d; ++k) {
                TTR_CUDA(cudaMemcpyAsync(t->core(b, k), host + b * tot + o, sizeof(double) * t->core_size(k),
                                         cudaMemcpyHostToDevice, ctx->c.stream));
                o += t->core_size(k);
            }
        }
        if (!all_finite(ctx->c, {{t->buf.p, static_cast<std::size_t>(t->stride * batch)}}))
            fail(Errc::InvalidArgument, "core entries must be finite");
        auto* o = new ttr_batch;
        o->t = std::move(t);
        *out = o;
    });
}

ttr_status ttr_batch_two_part_philox(ttr_ctx* ctx, int64_t batch, int64_t d, int64_t n, int64_t rx, int64_t rz,
                                     double eps, uint64_t seed, ttr_batch** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        need(batch >= 1 && d >= 2 && n >= 1 && rx >= 1 && rz >= 1, "bad batch shape");
        auto* o = new ttr_batch;
        o->t = batch_two_part_philox(ctx->c, batch, d, n, rx, rz, eps, seed);
        *out = o;
    });
}

ttr_status ttr_batch_shape(const ttr_batch* b, int64_t* batch, int64_t* d, int64_t* n, int64_t* r, int64_t* total) {
    return guard([&] {
        need(b && b->t, "null batch");
        const TTBatch& t = *b->t;
        if (batch) *batch = t.batch;
        if (d) *d = t.d();
        if (n) for (i64 k = 0; k < t.d(); ++k) n[k] = t.n[k];
        if (r) for (i64 k = 0; k <= t.d(); ++k) r[k] = t.r[k];
        if (total) *total = t.total();
    });
}

ttr_status ttr_batch_download(ttr_ctx* ctx, const ttr_batch* b, int64_t first, int64_t count, double* host) {
    return guard_ctx(ctx, [&] {
        need(ctx && b && b->t && host, "null argument");
        const TTBatch& t = *b->t;
        if (first < 0 || count < 0 || first + count > t.batch) fail(Errc::IndexOutOfRange, "batch range out of range");
        const i64 tot = t.total();
        for (i64 q = 0; q < count; ++q) {
            i64 o = 0;
            for (i64 k = 0; k < t.d(); ++k) {
                TTR_CUDA(cudaMemcpyAsync(host + q * tot + o, t.core(first + q, k), sizeof(double) * t.core_size(k),
                                         cudaMemcpyDeviceToHost, ctx->c.stream));
                o += t.core_size(k);
            }
        }
        TTR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

ttr_status ttr_batch_destroy(ttr_batch* b) {
    return guard([&] { delete b; });
}

ttr_status ttr_round_fixed_krp_batched(ttr_ctx* ctx, const ttr_batch* b, const int64_t* ranks, int64_t count,
                                       uint64_t seed, ttr_batch** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && b && b->t && out, "null argument");
        if (count < 0 || (count > 0 && !ranks)) fail(Errc::InvalidRanks, "expected d-1 target ranks");
        auto* o = new ttr_batch;
        o->t = round_fixed_krp_batched(ctx->c, *b->t, vec(ranks, count), seed);
        *out = o;
    });
}

ttr_status ttr_counters(ttr_ctx* ctx, ttr_counts* out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        out->gemm = ctx->c.counts.gemm;
        out->qr = ctx->c.counts.qr;
        out->svd = ctx->c.counts.svd;
        out->sketch = ctx->c.counts.sketch;
        out->rng = ctx->c.counts.rng;
    });
}

ttr_status ttr_counters_reset(ttr_ctx* ctx) {
    return guard_ctx(ctx, [&] {
        need(ctx != nullptr, "null context");
        ctx->c.counts = Counts{};
    });
}

}  // extern "C"

// ---- TT-GMRES cookie harness (tt_gmres.cu) ----
ttr_status ttr_kron_op_create(ttr_ctx* ctx, int64_t nterms, int64_t d, const int64_t* n, const double* factors,
                              ttr_kron_op** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && n && factors && out, "null argument");
        need(d >= 1 && nterms >= 1, "operator needs at least one term and one factor");
        auto* o = new ttr_kron_op;
        try {
            o->op = std::make_unique<KronOpDev>(ctx->c, nterms, vec(n, d), factors);
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

ttr_status ttr_kron_op_destroy(ttr_kron_op* op) {
    delete op;
    return TTR_OK;
}

ttr_status ttr_kron_op_shape(const ttr_kron_op* op, int64_t* nterms, int64_t* d, int64_t* n) {
    return guard([&] {
        need(op && op->op && nterms && d, "null argument");
        *nterms = op->op->nterms;
        *d = static_cast<int64_t>(op->op->n.size());
        if (n)
            for (std::size_t k = 0; k < op->op->n.size(); ++k) n[k] = op->op->n[k];
    });
}

ttr_status ttr_kron_op_factors(const ttr_kron_op* op, double* factors) {
    return guard([&] {
        need(op && op->op && factors, "null argument");
        std::size_t off = 0;
        for (const auto& term : op->op->host)
            for (const auto& a : term) {
                std::memcpy(factors + off, a.data(), sizeof(double) * a.size());
                off += a.size();
            }
    });
}

ttr_status ttr_cookie_problem(ttr_ctx* ctx, int64_t num_param_modes, int64_t grid_size, int64_t num_param_samples,
                              double rho_min, double rho_max, ttr_kron_op** op, ttr_tt** rhs) {
    return guard_ctx(ctx, [&] {
        need(ctx && op && rhs, "null argument");
        std::unique_ptr<TTDev> b;
        auto k = cookie_problem(ctx->c, num_param_modes, grid_size, num_param_samples, rho_min, rho_max, &b);
        auto* o = new ttr_kron_op;
        o->op = std::move(k);
        *op = o;
        *rhs = wrap(std::move(b));
    });
}

ttr_status ttr_apply_operator(ttr_ctx* ctx, const ttr_kron_op* op, const ttr_tt* x, ttr_tt** out_terms) {
    return guard_ctx(ctx, [&] {
        need(ctx && op && op->op && x && x->t && out_terms, "null argument");
        auto terms = apply_operator(ctx->c, *op->op, *x->t);
        for (std::size_t i = 0; i < terms.size(); ++i) out_terms[i] = wrap(std::move(terms[i]));
    });
}

ttr_status ttr_tt_gmres(ttr_ctx* ctx, const ttr_kron_op* op, const ttr_tt* rhs, const ttr_gmres_cfg* cfg,
                        ttr_gmres_result* result, ttr_tt** solution) {
    return guard_ctx(ctx, [&] {
        need(ctx && op && op->op && rhs && rhs->t && cfg && result && solution, "null argument");
        need(result->residual_history && result->max_rank_history, "history buffers are required");
        need(cfg->strategy >= TTR_GMRES_DETERMINISTIC && cfg->strategy <= TTR_GMRES_ADAPTIVE_KRP_SUM,
             "unknown rounding strategy");
        auto r = tt_gmres(ctx->c, *op->op, *rhs->t, *cfg);
        result->iterations = r.iterations;
        result->converged = r.converged ? 1 : 0;
        result->rounding_seconds = r.rounding_seconds;
        for (std::size_t i = 0; i < r.residual_history.size(); ++i) result->residual_history[i] = r.residual_history[i];
        for (std::size_t i = 0; i < r.max_rank_history.size(); ++i) result->max_rank_history[i] = r.max_rank_history[i];
        if (result->true_residual_history)
            for (std::size_t i = 0; i < r.true_residual_history.size(); ++i)
                result->true_residual_history[i] = r.true_residual_history[i];
        if (result->rounding_seconds_history)
            for (std::size_t i = 0; i < r.rounding_seconds_history.size(); ++i)
                result->rounding_seconds_history[i] = r.rounding_seconds_history[i];
        *solution = wrap(std::move(r.solution));
    });
}
