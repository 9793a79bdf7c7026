// sketch.cuh — device KRP sketch state shared by the rounding drivers
// (tt_round.cu, tt_sum.cu).
#pragma once

#include "common.cuh"
#include "rng_host.h"
#include "tt_round.h"

namespace ttr {

// KRP sketch state — sketch.cpp:44-92. Factors and contractions of modes
// start..d with a column capacity so that adaptive appends are in place.
struct Sketch {
    Ctx& c;
    const TTDev& t;
    i64 cap, cols = 0;
    std::vector<DBuf> omega;  // index k (1-based mode), n_k x cap, ld ldo[k]
    std::vector<i64> ldo;
    std::vector<DBuf> W;      // r_{k-1} x cap, ld ldw[k]
    std::vector<i64> ldw;
    std::vector<DBuf> Wt;     // cap x r_{k-1}, ld cap_even
    i64 ldwt;
    DBuf ones;
    std::vector<i64> width;   // current column count per mode
    std::vector<i64> charged; // columns per mode the reference's appends would have made (charges)
    int rng_mode;
    std::uint64_t seed;
    XoshiroGauss xo;

    Sketch(Ctx& cc, const TTDev& tt, i64 capacity, int mode, std::uint64_t s)
        : c(cc), t(tt), cap(capacity), rng_mode(mode), seed(s), xo(s) {
        const i64 d = t.d();
        omega.resize(d + 1);
        W.resize(d + 1);
        Wt.resize(d + 2);
        ldo.assign(d + 1, 0);
        ldw.assign(d + 1, 0);
        width.assign(d + 2, 0);
        charged.assign(d + 2, 0);
        ldwt = even_ld(cap);
        for (i64 k = 2; k <= d; ++k) {
            ldo[k] = even_ld(t.n[k - 1]);
            omega[k] = DBuf(c, static_cast<std::size_t>(ldo[k] * cap));
            ldw[k] = even_ld(t.r[k - 1]);
            W[k] = DBuf(c, static_cast<std::size_t>(ldw[k] * cap));
            if (k >= 3) Wt[k] = DBuf(c, static_cast<std::size_t>(ldwt * t.r[k - 1]));
        }
        ones = DBuf(c, static_cast<std::size_t>(ldwt));
        fill(c, ones.p, static_cast<std::size_t>(ldwt), 1.0);
    }

    // Draw `extra` fresh columns for modes start..d (draw_gaussian_factors,
    // sketch.cpp:44-56, in the reference's order) and contract them
    // (contract_tail, sketch.cpp:29-40), appending to W_start..W_d.
    void append(i64 start, i64 extra) {
        const i64 d = t.d();
        const i64 col0 = width[d];
        if (col0 + extra > cap) throw Error(TTR_ERR_INTERNAL, "sketch capacity exceeded");
        for (i64 k = start; k <= d; ++k) {
            const i64 nk = t.n[k - 1];
            double* dst = omega[k].p + col0 * ldo[k];
            if (rng_mode == TTR_RNG_PHILOX) {
                philox_factor(c, seed, k, nk, extra, col0, dst, ldo[k]);
            } else {
                auto host = xo.matrix(nk, extra);
                c.counts.rng += static_cast<std::uint64_t>(nk * extra);
                for (i64 j = 0; j < extra; ++j)
                    TTR_CUDA(cudaMemcpyAsync(dst + j * ldo[k], host.data() + j * nk, sizeof(double) * nk,
                                             cudaMemcpyHostToDevice, c.stream));
                TTR_CUDA(cudaStreamSynchronize(c.stream));  // host staging buffer lifetime
            }
        }
        SketchScope scope(c);
        for (i64 k = d; k >= start; --k) {
            const i64 rl = t.r[k - 1], nk = t.n[k - 1], rr = t.r[k];
            if (c.io) c.io->wait_in(c.stream, static_cast<std::size_t>(k - 1));  // core k-1 arrived (H2D)
            // Wt only carries this append's columns to the next mode: it starts
            // at column 0 so the contraction's W operand is always 16-byte
            // aligned (TMA-eligible) whatever the append offset
            const double* wt_next = (k == d) ? ones.p : Wt[k + 1].p;
            const i64 ld_next = ldwt;
            double* wt_out = (k >= 3) ? Wt[k].p : nullptr;
            krp_step(c, rl, nk, rr, extra, t.core(k - 1), omega[k].p + col0 * ldo[k], ldo[k], k == d ? ones.p : wt_next,
                     ld_next, W[k].p + col0 * ldw[k], ldw[k], wt_out, ldwt, k == d);
            width[k] = col0 + extra;
            charged[k] = width[k];
        }
    }

    // Make W_start..W_d hold at least `target` columns (the adaptive residual
    // sketch, round_rand.cpp:88-91: the reference appends exactly the missing
    // columns). With the counter-based Philox factors a column does not depend
    // on when or with which others it is contracted (bitwise: append ==
    // one-shot), so the device appends at least `chunk` columns at a time —
    // fewer passes over the cores — while the counters are charged exactly as
    // the reference's appends would be, when the columns are first used.
    void ensure(i64 start, i64 target, i64 chunk) {
        const i64 d = t.d();
        if (rng_mode != TTR_RNG_PHILOX) {
            if (width[start] < target) append(start, target - width[start]);
            return;
        }
        if (width[start] < target) {
            const i64 extra = std::min(std::max(target - width[start], chunk), cap - width[d]);
            const Counts saved = c.counts;
            const std::vector<i64> keep = charged;
            append(start, std::max(extra, target - width[start]));
            c.counts = saved;  // charged below, as the reference would
            charged = keep;
        }
        for (i64 k = start; k <= d; ++k) {
            if (charged[k] >= target) continue;
            const i64 cols = target - charged[k];
            const std::uint64_t rl = t.r[k - 1], nk = t.n[k - 1], rr = t.r[k];
            c.counts.rng += nk * static_cast<std::uint64_t>(cols);
            const std::uint64_t f = (k == d) ? 2ULL * rl * nk * cols : cols * (2ULL * rr * rl * nk + 2ULL * rl * rr);
            c.counts.gemm += f;
            c.counts.sketch += f;
            charged[k] = target;
        }
    }
};

// The same state for a batch of identically shaped TT tensors sharing ONE
// factor draw (sum of TT tensors, tt_sum.cu): the per-term contractions are
// stored STACKED, W_k = [W_k^(1); ...; W_k^(s)] ((s r_{k-1}) x cap), so the
// sketch of the sum  sum_i V_i W^(i)  is one GEMM with the concatenated V, and
// each append is one strided-batch KRP step per mode for all terms.
struct BatchSketch {
    Ctx& c;
    const TTBatch& t;
    i64 cap, s;
    std::vector<DBuf> omega;  // n_k x cap, shared by the terms
    std::vector<i64> ldo;
    std::vector<DBuf> W;      // (s r_{k-1}) x cap, ld ldw[k] = s r_{k-1}
    std::vector<i64> ldw;
    std::vector<DBuf> Wt;     // per term cap x r_{k-1} (ld ldwt), term stride ldwt r_{k-1}
    i64 ldwt;
    DBuf ones;
    std::vector<i64> width;
    std::vector<i64> charged;  // Sketch::charged
    int rng_mode;
    std::uint64_t seed;
    XoshiroGauss xo;

    BatchSketch(Ctx& cc, const TTBatch& tt, i64 capacity, int mode, std::uint64_t sd)
        : c(cc), t(tt), cap(capacity), s(tt.batch), rng_mode(mode), seed(sd), xo(sd) {
        const i64 d = t.d();
        omega.resize(d + 1);
        W.resize(d + 1);
        Wt.resize(d + 2);
        ldo.assign(d + 1, 0);
        ldw.assign(d + 1, 0);
        width.assign(d + 2, 0);
        charged.assign(d + 2, 0);
        ldwt = even_ld(cap);
        for (i64 k = 2; k <= d; ++k) {
            ldo[k] = even_ld(t.n[k - 1]);
            omega[k] = DBuf(c, static_cast<std::size_t>(ldo[k] * cap));
            ldw[k] = s * t.r[k - 1];
            W[k] = DBuf(c, static_cast<std::size_t>(ldw[k] * cap));
            if (k >= 3) Wt[k] = DBuf(c, static_cast<std::size_t>(ldwt * t.r[k - 1] * s));
        }
        ones = DBuf(c, static_cast<std::size_t>(ldwt));
        fill(c, ones.p, static_cast<std::size_t>(ldwt), 1.0);
    }

    void append(i64 start, i64 extra) {  // Sketch::append for all terms at once
        const i64 d = t.d();
        const i64 col0 = width[d];
        if (col0 + extra > cap) throw Error(TTR_ERR_INTERNAL, "sketch capacity exceeded");
        for (i64 k = start; k <= d; ++k) {
            const i64 nk = t.n[k - 1];
            double* dst = omega[k].p + col0 * ldo[k];
            if (rng_mode == TTR_RNG_PHILOX) {
                philox_factor(c, seed, k, nk, extra, col0, dst, ldo[k]);
            } else {
                auto host = xo.matrix(nk, extra);
                c.counts.rng += static_cast<std::uint64_t>(nk * extra);
                for (i64 j = 0; j < extra; ++j)
                    TTR_CUDA(cudaMemcpyAsync(dst + j * ldo[k], host.data() + j * nk, sizeof(double) * nk,
                                             cudaMemcpyHostToDevice, c.stream));
                TTR_CUDA(cudaStreamSynchronize(c.stream));
            }
        }
        SketchScope scope(c);
        for (i64 k = d; k >= start; --k) {
            const i64 rl = t.r[k - 1], nk = t.n[k - 1], rr = t.r[k];
            const bool last = (k == d);
            krp_step_batched(c, rl, nk, rr, extra, t.core(0, k - 1), t.stride, omega[k].p + col0 * ldo[k], ldo[k], 0,
                             last ? ones.p : Wt[k + 1].p, ldwt, last ? 0 : ldwt * rr, W[k].p + col0 * ldw[k],
                             ldw[k], rl, k >= 3 ? Wt[k].p : nullptr, ldwt, ldwt * rl, s, last);
            width[k] = col0 + extra;
            charged[k] = width[k];
        }
    }

    // Sketch::ensure for all terms (one shared factor draw, s contractions per mode)
    void ensure(i64 start, i64 target, i64 chunk) {
        const i64 d = t.d();
        if (rng_mode != TTR_RNG_PHILOX) {
            if (width[start] < target) append(start, target - width[start]);
            return;
        }
        if (width[start] < target) {
            const i64 extra = std::min(std::max(target - width[start], chunk), cap - width[d]);
            const Counts saved = c.counts;
            const std::vector<i64> keep = charged;
            append(start, std::max(extra, target - width[start]));
            c.counts = saved;
            charged = keep;
        }
        for (i64 k = start; k <= d; ++k) {
            if (charged[k] >= target) continue;
            const i64 cols = target - charged[k];
            const std::uint64_t rl = t.r[k - 1], nk = t.n[k - 1], rr = t.r[k];
            c.counts.rng += nk * static_cast<std::uint64_t>(cols);
            const std::uint64_t f = (k == d) ? 2ULL * rl * nk * cols : cols * (2ULL * rr * rl * nk + 2ULL * rl * rr);
            c.counts.gemm += f * static_cast<std::uint64_t>(s);
            c.counts.sketch += f * static_cast<std::uint64_t>(s);
            charged[k] = target;
        }
    }
};

}  // namespace ttr
