// tt_batch.cu — batched fixed-rank KRP rounding of many independent,
// identically shaped TT tensors (BASELINE config 5a: 4096 tensors, d=8, n=16,
// formal ranks 64, l=20). One launch per step covers the whole batch: the KRP
// sketch and every GEMM run as strided batches (grid.z = tensor), the QRs as
// one-CTA-per-matrix shared-memory Householder QR. Tensor b is rounded exactly
// as round_fixed_krp(Y_b, targets, derive_seed(seed, b)) in Philox mode.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "rng_host.h"
#include "tt_round.h"

namespace ttr {
namespace {
#include "qr_batch.cuh"
#include "lr_batch.cuh"

// Fused H(Y) = M H(X) + S_next = V(Y) W (lr_batch.cuh) when the shapes fit one
// CTA per tensor; false = caller takes the two-GEMM path.
// with_qr: also Q = qr(S) into a.Q and M_next = Q^T V(Y) into a.Mn (the
// per-tensor QR of the next step and its M GEMM fused into the same CTA; l n
// <= 320 and 17 <= l2 <= 24, else false)
bool lr_fused_qr_batched(Ctx& c, const lrb::LrArgs& a, i64 batch) {
    if (a.l > 24 || a.l2 > 24 || a.l2 < 17 || a.cols > 64 || a.rr > 64 || (a.cols & 1) || a.l < 1) return false;
    if (static_cast<i64>(a.l) * a.n > 320) return false;
    if ((reinterpret_cast<std::uintptr_t>(a.X) & 15) || (a.sX & 1)) return false;
    // Opt-in (TTR_LR_QR=1): measured on B200 (config 5a, phase timing, 4096
    // tensors per launch) 1.73 ms per mode fused vs 1.65 ms for the separate
    // sweep + QR + M launches — the two co-resident CTAs reach their
    // latency-bound QR epilogues together, so it does not hide behind the
    // other's streaming.
    static const bool on = [] {
        const char* e = std::getenv("TTR_LR_QR");
        return e && e[0] == '1';
    }();
    if (!on) return false;
    const int lt = (a.l + 7) / 8;
    bool done = false;
    auto go = [&](auto t1) {
        constexpr int LT = decltype(t1)::value;
        if (done || lt != LT) return;
        auto kern = lrb::lr_fused_kernel<LT, 3, 10>;
        constexpr std::size_t smem = lrb::LrSmem<LT>::kBytes;
        static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
        if (first_on_device(configured)) {
            TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        }
        kern<<<static_cast<unsigned>(batch), lrb::kThreads, smem, c.stream>>>(a);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        done = true;
    };
    go(std::integral_constant<int, 1>{});
    go(std::integral_constant<int, 2>{});
    go(std::integral_constant<int, 3>{});
    return done;
}

bool lr_fused_batched(Ctx& c, const lrb::LrArgs& a, i64 batch) {
    if (a.l > 32 || a.l2 > 32 || a.cols > 64 || a.rr > 64 || (a.cols & 1) || a.l < 1 || a.l2 < 1) return false;
    if ((reinterpret_cast<std::uintptr_t>(a.X) & 15) || (a.sX & 1)) return false;
    static const bool off = [] {
        const char* e = std::getenv("TTR_LR_FUSED");  // experiments: 0 = two GEMMs
        return e && e[0] == '0';
    }();
    if (off) return false;
    const int lt = (a.l + 7) / 8, lt2 = (a.l2 + 7) / 8;
    bool done = false;
    auto go = [&](auto t1, auto t2) {
        constexpr int LT = decltype(t1)::value, LT2 = decltype(t2)::value;
        if (done || lt != LT || lt2 != LT2) return;
        auto kern = lrb::lr_fused_kernel<LT, LT2>;
        constexpr std::size_t smem = lrb::LrSmem<LT>::kBytes;
        static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
        if (first_on_device(configured)) {
            TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        }
        kern<<<static_cast<unsigned>(batch), lrb::kThreads, smem, c.stream>>>(a);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        done = true;
    };
    auto row = [&](auto t1) {
        go(t1, std::integral_constant<int, 1>{});
        go(t1, std::integral_constant<int, 2>{});
        go(t1, std::integral_constant<int, 3>{});
        go(t1, std::integral_constant<int, 4>{});
    };
    row(std::integral_constant<int, 1>{});
    row(std::integral_constant<int, 2>{});
    row(std::integral_constant<int, 3>{});
    row(std::integral_constant<int, 4>{});
    return done;
}
}  // namespace

TTBatch::TTBatch(Ctx& c, i64 batch_, const std::vector<i64>& n_, const std::vector<i64>& r_)
    : ctx(&c), n(n_), r(r_), batch(batch_) {
    const i64 d = static_cast<i64>(n.size());
    if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
    if (static_cast<i64>(r.size()) != d + 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
    if (r.front() != 1 || r.back() != 1) fail(Errc::BoundaryRankNotOne, "boundary TT ranks must be 1");
    if (batch < 1) fail(Errc::InvalidArgument, "batch must be >= 1");
    off.resize(d + 1);
    i64 o = 0;
    for (i64 k = 0; k < d; ++k) {
        if (r[k] < 1 || n[k] < 1 || r[k + 1] < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
        off[k] = o;
        o += round_up(r[k] * n[k] * r[k + 1], 32);
    }
    off[d] = o;
    stride = o;
    buf = DBuf(c, static_cast<std::size_t>(stride * batch));
}

i64 TTBatch::total() const {
    i64 t = 0;
    for (i64 k = 0; k < d(); ++k) t += core_size(k);
    return t;
}

// ---------------------------------------------------------------------------
std::unique_ptr<TTBatch> batch_two_part_philox(Ctx& c, i64 batch, i64 d, i64 n, i64 rx, i64 rz, double eps,
                                               std::uint64_t seed) {
    std::vector<i64> modes(d, n), kx(d + 1, rx), kz(d + 1, rz), ky(d + 1, rx + rz);
    kx.front() = kx.back() = kz.front() = kz.back() = ky.front() = ky.back() = 1;
    auto out = std::make_unique<TTBatch>(c, batch, modes, ky);
    for (i64 b = 0; b < batch; ++b) {
        const std::uint64_t sb = derive_seed(seed, static_cast<std::uint64_t>(b));
        auto x = random_philox_tt(c, modes, kx, derive_seed(sb, 1));
        auto z = random_philox_tt(c, modes, kz, derive_seed(sb, 2));
        scale_tt(c, *x, 1.0 / norm_exact(c, *x));
        scale_tt(c, *z, eps / norm_exact(c, *z));
        auto y = formal_sum(c, {x.get(), z.get()});
        for (i64 k = 0; k < d; ++k)
            TTR_CUDA(cudaMemcpyAsync(out->core(b, k), y->core(k), sizeof(double) * y->core_size(k),
                                     cudaMemcpyDeviceToDevice, c.stream));
    }
    return out;
}

std::unique_ptr<TTDev> batch_get(Ctx& c, const TTBatch& t, i64 b) {
    if (b < 0 || b >= t.batch) fail(Errc::IndexOutOfRange, "batch index out of range");
    auto out = std::make_unique<TTDev>(c, t.n, t.r);
    for (i64 k = 0; k < t.d(); ++k)
        TTR_CUDA(cudaMemcpyAsync(out->core(k), t.core(b, k), sizeof(double) * t.core_size(k), cudaMemcpyDeviceToDevice,
                                 c.stream));
    return out;
}

// ---------------------------------------------------------------------------
// round_rand.cpp:52-64 (+ rand_orth_sweep :26-44) over a strided batch
std::unique_ptr<TTBatch> round_fixed_krp_batched(Ctx& c, const TTBatch& t, const std::vector<i64>& targets,
                                                 std::uint64_t seed) {
    const i64 d = t.d(), B = t.batch;
    if (static_cast<i64>(targets.size()) != d - 1) fail(Errc::InvalidRanks, "expected d-1 target ranks");
    for (i64 l : targets)
        if (l < 1) fail(Errc::InvalidRanks, "target ranks must be >= 1");
    if (d == 1) fail(Errc::InvalidArgument, "batched rounding needs d >= 2");
    const i64 width = *std::max_element(targets.begin(), targets.end());
    std::vector<i64> r(d + 1, 1);
    for (i64 k = 1; k < d; ++k) r[k] = std::min({targets[k - 1], r[k - 1] * t.n[k - 1], t.r[k]});
    auto out = std::make_unique<TTBatch>(c, B, t.n, r);

    // The batch runs as G independent groups of tensors, each on its own side
    // stream, so that one group's latency-bound QR launches overlap another
    // group's HBM/DMMA-bound sketch and sweep kernels (results are per tensor,
    // identical to one group). TTR_BATCH_GROUPS overrides G (1 = one stream).
    static const int groups_env = [] {
        const char* e = std::getenv("TTR_BATCH_GROUPS");
        return e ? std::atoi(e) : 0;
    }();
    // (phase timing — bench.py's per-kernel roofline run — needs one stream)
    const i64 G = c.timing ? 1 : std::max<i64>(1, std::min<i64>(groups_env > 0 ? groups_env : (B >= 1024 ? 2 : 1), B));

    // Per-tensor QRs of the sweep by batched CholeskyQR2 / shifted CholeskyQR3
    // (K4e, qr_chol.cu) where the sketch is structurally full rank (wbound, as in
    // rand_orth_sweep) and the shape fits; a tensor whose factorisation broke
    // down is redone afterwards through round_fixed_krp with its own seed (the
    // Householder path). TTR_BATCH_CQR=0 keeps the batched Householder QR.
    static const int cqr_env = [] {
        const char* e = std::getenv("TTR_BATCH_CQR");
        return e ? std::atoi(e) : 1;
    }();
    std::vector<i64> wbound(static_cast<std::size_t>(d + 2), 0);
    wbound[d] = std::min({t.r[d - 1], t.n[d - 1], width});
    for (i64 k = d - 1; k >= 2; --k) wbound[k] = std::min({t.r[k - 1], width, t.n[k - 1] * wbound[k + 1]});
    auto cqr_mode = [&](i64 k) {
        const i64 rows = r[k - 1] * t.n[k - 1], l = r[k];
        return cqr_env == 1 && cholqr_small_fits(rows, l) && wbound[k + 1] >= l;
    };
    bool any_cqr = false;
    for (i64 k = 1; k < d; ++k) any_cqr = any_cqr || cqr_mode(k);
    DBuf flag_buf;
    int* flags = nullptr;
    if (any_cqr) {
        flag_buf = DBuf(c, static_cast<std::size_t>((B + 1) / 2));
        flags = reinterpret_cast<int*>(flag_buf.p);
        TTR_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * static_cast<std::size_t>(B), c.stream));
    }
    auto redo_broken = [&] {
        if (!any_cqr) return;
        std::vector<int> h(static_cast<std::size_t>(B));
        TTR_CUDA(cudaMemcpyAsync(h.data(), flags, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
        for (i64 b = 0; b < B; ++b) {
            if (!h[static_cast<std::size_t>(b)]) continue;
            auto one = batch_get(c, t, b);
            auto y = round_fixed_krp(c, *one, targets, derive_seed(seed, static_cast<std::uint64_t>(b)), TTR_RNG_PHILOX);
            for (i64 k = 0; k < d; ++k)
                TTR_CUDA(cudaMemcpyAsync(out->core(b, k), y->core(k), sizeof(double) * y->core_size(k),
                                         cudaMemcpyDeviceToDevice, c.stream));
        }
    };
    if (any_cqr) TTR_CUDA(cudaStreamSynchronize(c.stream));  // flags zeroed before the side streams start
    auto run_group = [&](i64 b0, i64 Bg) {

        // ---- sketch: W_k for k = d..2 (Omega_k drawn per tensor from derive_seed(seed, b)) ----
        const i64 ldwt = even_ld(width);
        std::vector<DBuf> W(d + 2), Wt(d + 2);
        std::vector<i64> ldw(d + 2, 0), sw(d + 2, 0), swt(d + 2, 0);
        DBuf ones(c, static_cast<std::size_t>(ldwt));
        fill(c, ones.p, static_cast<std::size_t>(ldwt), 1.0);
        {
            PhaseScope ph(c, kPhaseSketch);
            SketchScope scope(c);
            for (i64 k = d; k >= 2; --k) {
                const i64 rl = t.r[k - 1], nk = t.n[k - 1], rr = t.r[k];
                const i64 ldo = even_ld(nk), so = ldo * width;
                DBuf om(c, static_cast<std::size_t>(so * Bg));
                philox_factor_batched(c, seed, k, nk, width, om.p, ldo, so, Bg, b0);
                ldw[k] = even_ld(rl);
                sw[k] = ldw[k] * width;
                W[k] = DBuf(c, static_cast<std::size_t>(sw[k] * Bg));
                swt[k] = ldwt * rl;
                if (k >= 3) Wt[k] = DBuf(c, static_cast<std::size_t>(swt[k] * Bg));
                const bool last = (k == d);
                krp_step_batched(c, rl, nk, rr, width, t.core(b0, k - 1), t.stride, om.p, ldo, so, last ? ones.p : Wt[k + 1].p,
                                 ldwt, last ? 0 : swt[k + 1], W[k].p, ldw[k], sw[k], k >= 3 ? Wt[k].p : nullptr, ldwt, swt[k],
                                 Bg, last);
            }
        }

        // ---- left-to-right Rand-Orth sweep ----
        i64 max_work = 0, max_s = 0;
        for (i64 k = 1; k < d; ++k) {
            max_work = std::max(max_work, r[k] * t.n[k] * t.r[k + 1]);
            max_s = std::max(max_s, r[k - 1] * t.n[k - 1] * r[k]);
        }
        DBuf work(c, static_cast<std::size_t>(max_work * Bg));
        DBuf S(c, static_cast<std::size_t>(max_s * Bg));
        DBuf M(c, static_cast<std::size_t>(width * t.max_rank() * Bg)), M2(c, static_cast<std::size_t>(width * t.max_rank() * Bg));
        double* Mcur = M.p;   // M_k = Q_k^T V(Y_k)
        double* Mnext = M2.p;  // written by the fused QR epilogue for step k+1
        const double* v = t.core(b0, 0);
        i64 sv = t.stride;
        bool s_ready = false;  // S of this step already formed by the previous fused step
        bool q_ready = false;  // ... and its QR (the output core) and M as well
        for (i64 k = 1; k < d; ++k) {
            const i64 rows = r[k - 1] * t.n[k - 1], cols = t.r[k], l = r[k];
            if (!s_ready) {
                PhaseScope ph(c, kPhaseGemm);
                gemm_batched(c, false, rows, l, cols, 1.0, v, rows, sv, W[k + 1].p, ldw[k + 1], sw[k + 1], 0.0, S.p, rows,
                             rows * l, Bg);
            }
            if (!q_ready) {
                PhaseScope ph(c, kPhaseQr);
                c.charge_qr(4ULL * static_cast<std::uint64_t>(rows) * l * std::min(rows, l) * Bg);
                if (cqr_mode(k)) {
                    cholqr_small_batched(c, rows, l, S.p, rows, rows * l, out->core(b0, k - 1), rows, out->stride, Bg,
                                         flags + b0);
                } else if (rows * l <= 26000) {
                    qr_small_batched(c, rows, l, S.p, rows, rows * l, out->core(b0, k - 1), rows, out->stride, nullptr, 1, 0, Bg);
                } else {
                    const Counts keep = c.counts;
                    for (i64 b = 0; b < Bg; ++b)
                        thin_qr(c, rows, l, S.p + b * rows * l, rows, out->core(b0 + b, k - 1), rows, nullptr, 1);
                    c.counts = keep;
                }
            }
            const i64 ncols = t.n[k] * t.r[k + 1];
            double* dst = (k == d - 1) ? out->core(b0, d - 1) : work.p;
            const i64 sdst = (k == d - 1) ? out->stride : l * ncols;
            if (!q_ready) {
                PhaseScope ph(c, kPhaseGemm);
                gemm_batched(c, true, l, cols, rows, 1.0, out->core(b0, k - 1), rows, out->stride, v, rows, sv, 0.0, Mcur, l,
                             l * cols, Bg);
            }
            {
                s_ready = false;
                q_ready = false;
                if (k < d - 1) {
                    PhaseScope ph(c, kPhaseOther);  // the fused kernel alone (bench.py roofline)
                    // next step's sketch S = V(Y_{k+1}) W_{k+2} fused with Y_{k+1} = M H(X_{k+1})
                    lrb::LrArgs a{};
                    a.l = static_cast<int>(l);
                    a.cols = static_cast<int>(cols);
                    a.n = static_cast<int>(t.n[k]);
                    a.rr = static_cast<int>(t.r[k + 1]);
                    a.l2 = static_cast<int>(r[k + 1]);
                    a.M = Mcur;
                    a.sM = l * cols;
                    a.X = t.core(b0, k);
                    a.sX = t.stride;
                    a.W = W[k + 2].p;
                    a.ldw = ldw[k + 2];
                    a.sW = sw[k + 2];
                    a.Y = dst;
                    a.sY = sdst;
                    a.S = S.p;
                    a.sS = l * t.n[k] * r[k + 1];
                    // ... and, when the shapes allow, step k+1's QR (output core k+1)
                    // and M_{k+1} = Q^T V(Y_{k+1}) in the same CTA
                    const i64 rows2 = l * t.n[k], l2 = r[k + 1], cols2 = t.r[k + 1];
                    a.Q = out->core(b0, k);
                    a.sQ = out->stride;
                    a.Mn = Mnext;
                    a.sMn = l2 * cols2;
                    q_ready = lr_fused_qr_batched(c, a, Bg);
                    s_ready = q_ready || lr_fused_batched(c, a, Bg);
                    if (s_ready) {
                        c.charge_gemm(2ULL * static_cast<std::uint64_t>(l) * ncols * cols * Bg);
                        c.charge_gemm(2ULL * static_cast<std::uint64_t>(l * t.n[k]) * r[k + 1] * t.r[k + 1] * Bg);
                    }
                    if (q_ready) {
                        c.charge_qr(4ULL * static_cast<std::uint64_t>(rows2) * l2 * std::min(rows2, l2) * Bg);
                        c.charge_gemm(2ULL * static_cast<std::uint64_t>(l2) * cols2 * rows2 * Bg);
                        std::swap(Mcur, Mnext);
                    }
                }
                if (!s_ready) {
                    PhaseScope ph(c, kPhaseGemm);
                    gemm_batched(c, false, l, ncols, cols, 1.0, Mcur, l, l * cols, t.core(b0, k), cols, t.stride, 0.0, dst, l,
                                 sdst, Bg);
                }
            }
            v = dst;
            sv = sdst;
        }
    };
    if (G == 1) {
        run_group(0, B);
        redo_broken();
        return out;
    }
    c.fork_side(static_cast<int>(G));
    const cudaStream_t main = c.stream;
    double* const main_work = c.work;
    const std::size_t main_bytes = c.work_bytes;
    const bool timing = c.timing;
    c.timing = false;  // per-phase events would time interleaved streams
    std::vector<double*> works;
    auto restore = [&] {
        c.stream = main;
        c.work = main_work;
        c.work_bytes = main_bytes;
        c.timing = timing;
    };
    try {
        for (i64 g = 0; g < G; ++g) {
            const i64 b0 = B * g / G, b1 = B * (g + 1) / G;
            c.stream = c.side[g];
            c.work = nullptr;
            c.work_bytes = 0;
            run_group(b0, b1 - b0);
            if (c.work) works.push_back(c.work);
        }
    } catch (...) {
        restore();
        throw;
    }
    restore();
    c.join_side(static_cast<int>(G));
    for (double* w : works) TTR_CUDA(cudaFreeAsync(w, c.stream));
    redo_broken();
    return out;
}

}  // namespace ttr
