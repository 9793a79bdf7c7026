// tt_sum.cu — adaptive randomized rounding of a SUM of TT tensors without
// forming the formal sum (proj/core/src/sum_round.cpp:21-173, Alg. 11 of the
// paper): one shared Gaussian factor draw, one KRP sketch per term (K2 on each
// term's own cores — the formal sum's block-diagonal zeros are never touched),
// and a working unfolding V that keeps one column block per term. The sketch
// of the sum is the sum of the per-term sketches, accumulated by GEMMs with
// beta = 1; every other step is the single-tensor adaptive loop of
// round_adaptive_krp on the concatenated V.
#include <algorithm>
#include <cmath>
#include <limits>

#include "common.cuh"
#include "sketch.cuh"
#include "tt_round.h"

namespace ttr {

static i64 ceil_frac(double f, i64 n) {  // round_rand.cpp:46-48
    return std::max<i64>(1, static_cast<i64>(std::ceil(f * static_cast<double>(n))));
}

std::unique_ptr<TTDev> round_sum_adaptive_krp(Ctx& c, const std::vector<const TTDev*>& terms, double eps, double f_inc,
                                              std::uint64_t seed, int rng_mode) {
    if (terms.empty()) fail(Errc::EmptyTermList, "sum of no TT terms");  // sum_round.cpp:11-19
    const auto& modes = terms.front()->n;
    for (const TTDev* t : terms)
        if (t->n != modes) fail(Errc::ModeSizeMismatch, "sum terms mode sizes differ");
    if (!(eps > 0.0)) fail(Errc::InvalidArgument, "tolerance must be > 0");
    if (!(f_inc > 0.0 && f_inc < 1.0)) fail(Errc::InvalidArgument, "f_inc must lie in (0,1)");
    const i64 s_count = static_cast<i64>(terms.size());
    const i64 d = static_cast<i64>(modes.size());
    if (d == 1) {  // the sum is exact at rank one
        auto out = std::make_unique<TTDev>(c, modes, std::vector<i64>{1, 1});
        TTR_CUDA(cudaMemsetAsync(out->core(0), 0, sizeof(double) * modes[0], c.stream));
        for (const TTDev* t : terms) axpy_matrix(c, modes[0], 1, 1.0, t->core(0), modes[0], out->core(0), modes[0]);
        return out;
    }
    i64 width = 1, rsum = 0;
    for (const TTDev* t : terms) {
        width = std::max(width, t->max_rank());
        rsum += t->max_rank();
    }
    // column capacity of every term's sketch: rbar <= sum of the term ranks
    const i64 cap = std::max(width, rsum + ceil_frac(f_inc, rsum) + 1);
    // Identically shaped terms (e.g. the 20 terms of config 4) run batched:
    // one stacked sketch (BatchSketch), the sketch of the sum as ONE GEMM, the
    // next working unfolding as one strided-batch GEMM. Otherwise one Sketch
    // per term (same seed and draw sequence: the shared factor draw).
    bool same = true;
    for (const TTDev* t : terms) same = same && t->r == terms.front()->r;
    std::unique_ptr<TTBatch> tb;
    std::unique_ptr<BatchSketch> bsk;
    std::vector<std::unique_ptr<Sketch>> sk;
    if (same && s_count > 1) {
        tb = std::make_unique<TTBatch>(c, s_count, modes, terms.front()->r);
        for (i64 i = 0; i < s_count; ++i)
            for (i64 k = 0; k < d; ++k)
                TTR_CUDA(cudaMemcpyAsync(tb->core(i, k), terms[i]->core(k), sizeof(double) * tb->core_size(k),
                                         cudaMemcpyDeviceToDevice, c.stream));
        bsk = std::make_unique<BatchSketch>(c, *tb, cap, rng_mode, seed);
        bsk->append(2, width);
    } else {
        for (const TTDev* t : terms) {
            sk.push_back(std::make_unique<Sketch>(c, *t, cap, rng_mode, seed));
            sk.back()->append(2, width);
        }
    }
    // W_k^(i)(:, col0:) of term i
    auto w_of = [&](i64 i, i64 k, i64 col0) -> std::pair<const double*, i64> {
        if (bsk) return {bsk->W[k].p + i * terms[i]->r[k - 1] + col0 * bsk->ldw[k], bsk->ldw[k]};
        return {sk[i]->W[k].p + col0 * sk[i]->ldw[k], sk[i]->ldw[k]};
    };
    // norm estimate of the sum from the initial sketches (sum_round.cpp:78-91)
    const i64 n0 = modes[0];
    DBuf S0(c, static_cast<std::size_t>(n0 * width)), Si(c, static_cast<std::size_t>(n0 * width));
    TTR_CUDA(cudaMemsetAsync(S0.p, 0, sizeof(double) * n0 * width, c.stream));
    double max_term = 0.0;
    for (i64 i = 0; i < s_count; ++i) {
        const TTDev& t = *terms[i];
        auto w2 = w_of(i, 2, 0);
        gemm(c, false, n0, width, t.r[1], 1.0, t.core(0), n0, w2.first, w2.second, 0.0, Si.p, n0);
        max_term = std::max(max_term, frob_norm(c, n0, width, Si.p, n0) / std::sqrt(static_cast<double>(width)));
        axpy_matrix(c, n0, width, 1.0, Si.p, n0, S0.p, n0);
    }
    const double nrm = frob_norm(c, n0, width, S0.p, n0) / std::sqrt(static_cast<double>(width));
    if (nrm < 1e3 * std::numeric_limits<double>::epsilon() * max_term) {  // cancellation: the zero tensor
        auto z = std::make_unique<TTDev>(c, modes, std::vector<i64>(static_cast<std::size_t>(d + 1), 1));
        TTR_CUDA(cudaMemsetAsync(z->buf.p, 0, sizeof(double) * z->off.back(), c.stream));
        return z;
    }
    const double tau = eps * nrm / std::sqrt(static_cast<double>(d - 1));

    // working unfolding V: rows x sum_i r_k^(i), one column block per term
    i64 max_rows = 0, max_v = 0;
    {
        i64 lp = 1;
        for (i64 k = 1; k < d; ++k) {
            i64 cols = 0, cols1 = 0;
            for (const TTDev* t : terms) {
                cols += t->r[k];
                cols1 += t->r[k + 1];
            }
            const i64 rows = lp * modes[k - 1];
            max_rows = std::max(max_rows, rows);
            max_v = std::max(max_v, rows * cols);
            lp = std::min(rows, cols);
            max_v = std::max(max_v, lp * modes[k] * cols1);  // the next working unfolding
        }
    }
    const i64 rcap = std::min(rsum, max_rows);
    DBuf vbuf(c, static_cast<std::size_t>(max_v + 1));
    DBuf vnext(c, static_cast<std::size_t>(max_v + 1));
    DBuf Qb(c, static_cast<std::size_t>(max_rows * (rcap + 1)));
    DBuf Sb(c, static_cast<std::size_t>(max_rows * cap));
    DBuf Qn(c, static_cast<std::size_t>(max_rows * cap));
    DBuf P(c, static_cast<std::size_t>(std::max<i64>(rcap, cap) * cap + 1));
    DBuf Mb(c, static_cast<std::size_t>((rcap + 1) * rsum + 1));
    // V(Y_1) = [V(X_1^(1)) V(X_1^(2)) ...]
    {
        i64 c0 = 0;
        for (const TTDev* t : terms) {
            copy_matrix(c, n0, t->r[1], t->core(0), n0, vbuf.p + c0 * n0, n0);
            c0 += t->r[1];
        }
    }
    std::vector<DBuf> out_cores;
    std::vector<i64> r_out(static_cast<std::size_t>(d + 1), 1);
    i64 l_prev = 1;
    DBuf last;
    for (i64 k = 1; k < d; ++k) {
        const i64 rows = l_prev * modes[k - 1];
        i64 vcols = 0;
        for (const TTDev* t : terms) vcols += t->r[k];
        const double* v = vbuf.p;  // rows x vcols, ld rows
        const i64 rbar = std::min(rows, vcols);
        i64 b_init = 1;
        for (const TTDev* t : terms) b_init = std::max(b_init, t->r[k]);
        b_init = std::min(b_init, rbar);
        // S = sum_i V_i W_{k+1}^(i)(:, cols) — the sketch of the sum
        auto sketch_into = [&](i64 col0, i64 ncols) {
            if (bsk) {  // V [W^(1); ...; W^(s)]: one GEMM
                gemm(c, false, rows, ncols, vcols, 1.0, v, rows, bsk->W[k + 1].p + col0 * bsk->ldw[k + 1],
                     bsk->ldw[k + 1], 0.0, Sb.p, rows);
                return;
            }
            i64 c0 = 0;
            for (i64 i = 0; i < s_count; ++i) {
                const i64 rk = terms[i]->r[k];
                auto wk = w_of(i, k + 1, col0);
                gemm(c, false, rows, ncols, rk, 1.0, v + c0 * rows, rows, wk.first, wk.second, i == 0 ? 0.0 : 1.0,
                     Sb.p, rows);
                c0 += rk;
            }
        };
        sketch_into(0, b_init);
        thin_qr(c, rows, b_init, Sb.p, rows, Qb.p, rows, nullptr, 1);
        i64 q = std::min(rows, b_init);
        const i64 ldm = rcap + 1;  // M = Q^T V (ld rcap+1), formed once after the growth loop
        const i64 b_inc = ceil_frac(f_inc, rbar);
        while (q < rbar) {
            // residual_sketch_sum (sum_round.cpp:21-50): one shared fresh draw
            // appends in chunks (Sketch::ensure; charges stay column-exact)
            const i64 chunk = 4 * ceil_frac(f_inc, rsum);
            if (bsk) {
                bsk->ensure(k + 1, q + b_inc, chunk);
            } else {
                for (i64 i = 0; i < s_count; ++i) sk[i]->ensure(k + 1, q + b_inc, chunk);
            }
            sketch_into(q, b_inc);
            gemm(c, true, q, b_inc, rows, 1.0, Qb.p, rows, Sb.p, rows, 0.0, P.p, q);
            gemm(c, false, rows, b_inc, q, -1.0, Qb.p, rows, P.p, q, 1.0, Sb.p, rows);
            const double est = frob_norm(c, rows, b_inc, Sb.p, rows) / std::sqrt(static_cast<double>(b_inc));
            if (est <= tau) break;
            const i64 grow = std::min(b_inc, rbar - q);
            growth_basis(c, rows, q, grow, Qb.p, Sb.p, Qn.p, P.p);
            q += grow;
        }
        gemm(c, true, q, vcols, rows, 1.0, Qb.p, rows, v, rows, 0.0, Mb.p, ldm);  // M = Q^T V
        DBuf core(c, static_cast<std::size_t>(rows * q));
        copy_matrix(c, rows, q, Qb.p, rows, core.p, rows);
        out_cores.push_back(std::move(core));
        r_out[k] = q;
        l_prev = q;
        // next working unfolding (or the last core): per-term M_i H(X_{k+1}^(i))
        const i64 nk1 = modes[k];
        if (k == d - 1) {
            last = DBuf(c, static_cast<std::size_t>(q * nk1));
            i64 c0 = 0;
            for (i64 i = 0; i < s_count; ++i) {
                const TTDev& t = *terms[i];
                gemm(c, false, q, nk1, t.r[k], 1.0, Mb.p + c0 * ldm, ldm, t.core(k), t.r[k], i == 0 ? 0.0 : 1.0,
                     last.p, q);
                c0 += t.r[k];
            }
        } else {
            const i64 rows1 = q * nk1;
            i64 c0 = 0, oc = 0;
            if (tb) {  // M_i H(X_{k+1}^(i)) for all terms: one strided-batch GEMM
                const i64 rk = tb->r[k], rk1 = tb->r[k + 1];
                gemm_batched(c, false, q, nk1 * rk1, rk, 1.0, Mb.p, ldm, rk * ldm, tb->core(0, k), rk, tb->stride, 0.0,
                             vnext.p, q, rows1 * rk1, s_count);
                std::swap(vbuf, vnext);
                continue;
            }
            for (i64 i = 0; i < s_count; ++i) {
                const TTDev& t = *terms[i];
                // the horizontal product (q x n r_{k+1}) is the next vertical block (q n x r_{k+1})
                gemm(c, false, q, nk1 * t.r[k + 1], t.r[k], 1.0, Mb.p + c0 * ldm, ldm, t.core(k), t.r[k], 0.0,
                     vnext.p + oc * rows1, q);
                c0 += t.r[k];
                oc += t.r[k + 1];
            }
            std::swap(vbuf, vnext);
        }
    }
    auto out = std::make_unique<TTDev>(c, modes, r_out);
    for (i64 k = 0; k < d - 1; ++k)
        copy_matrix(c, out->core_size(k), 1, out_cores[k].p, out->core_size(k), out->core(k), out->core_size(k));
    copy_matrix(c, out->core_size(d - 1), 1, last.p, out->core_size(d - 1), out->core(d - 1), out->core_size(d - 1));
    return out;
}

}  // namespace ttr
