// tt_det.cu — deterministic TT-SVD rounding (the comparison path), on device:
// round_deterministic (proj/core/src/orthogonalize.cpp:117-140) = right-to-left
// orthogonalisation (:13-26) + left-to-right compression sweep (:44-58) with
// truncated SVDs (:87-115).
#include <algorithm>
#include <cmath>
#include <limits>

#include "common.cuh"
#include "tt_round.h"

namespace ttr {
namespace {

// Truncation rule of orthogonalize.cpp:87-115 on host singular values.
i64 truncation_rank(const std::vector<double>& s, i64 rows, i64 cols, bool tol_rule, double tau, i64 l) {
    const i64 count = static_cast<i64>(s.size());
    i64 keep;
    if (tol_rule) {
        const double floor = count > 0 ? s[0] * static_cast<double>(std::max(rows, cols)) *
                                             std::numeric_limits<double>::epsilon()
                                       : 0.0;
        const double t = std::max(tau, floor);
        double tail = 0.0;
        keep = count;
        while (keep > 1) {
            const double cand = tail + s[keep - 1] * s[keep - 1];
            if (std::sqrt(cand) > t) break;
            tail = cand;
            --keep;
        }
    } else {
        keep = std::min(l, count);
    }
    return std::max<i64>(keep, 1);
}

std::unique_ptr<TTDev> compress_sweep(Ctx& c, const TTDev& right_orth, bool tol_rule, double tau,
                                      const std::vector<i64>* ranks) {
    const i64 d = right_orth.d();
    const auto& n = right_orth.n;
    std::vector<i64> r = right_orth.r;
    std::vector<DBuf> cores(d);
    // work = current core k (grows), starting with core 0
    i64 max_core = 0, maxr = right_orth.max_rank();
    for (i64 k = 0; k < d; ++k) max_core = std::max(max_core, right_orth.core_size(k));
    DBuf cur(c, static_cast<std::size_t>(max_core));
    copy_matrix(c, right_orth.core_size(0), 1, right_orth.core(0), right_orth.core_size(0), cur.p, right_orth.core_size(0));
    DBuf Q(c, static_cast<std::size_t>(max_core));
    DBuf R(c, static_cast<std::size_t>(maxr * maxr));
    DBuf U(c, static_cast<std::size_t>(maxr * maxr));
    DBuf SV(c, static_cast<std::size_t>(maxr * maxr));
    std::vector<double> s;
    for (i64 k = 0; k + 1 < d; ++k) {
        const i64 rl = r[k], rows = rl * n[k], rr = r[k + 1], kk = std::min(rows, rr);
        thin_qr(c, rows, rr, cur.p, rows, Q.p, rows, R.p, kk);
        svd_left(c, kk, rr, R.p, kk, U.p, kk, s, nullptr);
        const i64 keep = truncation_rank(s, kk, rr, tol_rule, tau, ranks ? (*ranks)[k] : 0);
        // core k = Q U(:, 1:keep)
        cores[k] = DBuf(c, static_cast<std::size_t>(rows * keep));
        gemm(c, false, rows, keep, kk, 1.0, Q.p, rows, U.p, kk, 0.0, cores[k].p, rows);
        // SV = diag(s) V^T (keep x rr) = U(:, 1:keep)^T R; next core = SV H(core_{k+1})
        gemm(c, true, keep, rr, kk, 1.0, U.p, kk, R.p, kk, 0.0, SV.p, keep);
        const i64 ncols = n[k + 1] * r[k + 2];
        gemm(c, false, keep, ncols, rr, 1.0, SV.p, keep, right_orth.core(k + 1), rr, 0.0, cur.p, keep);
        r[k + 1] = keep;
    }
    auto out = std::make_unique<TTDev>(c, n, r);
    for (i64 k = 0; k + 1 < d; ++k)
        copy_matrix(c, out->core_size(k), 1, cores[k].p, out->core_size(k), out->core(k), out->core_size(k));
    copy_matrix(c, out->core_size(d - 1), 1, cur.p, out->core_size(d - 1), out->core(d - 1), out->core_size(d - 1));
    return out;
}

}  // namespace

std::unique_ptr<TTDev> round_deterministic_tol(Ctx& c, const TTDev& t, double eps) {  // orthogonalize.cpp:117-127
    if (eps < 0) fail(Errc::InvalidArgument, "rounding tolerance must be >= 0");
    const i64 d = t.d();
    if (d == 1) return copy_tt(c, t);
    auto o = orthogonalize_rl_public(c, t);
    const double nrm = frob_norm(c, o->core_size(0), 1, o->core(0), o->core_size(0));
    const double tau = eps * nrm / std::sqrt(static_cast<double>(d - 1));
    return compress_sweep(c, *o, true, tau, nullptr);
}

std::unique_ptr<TTDev> round_deterministic_ranks(Ctx& c, const TTDev& t, const std::vector<i64>& ranks) {  // :129-140
    const i64 d = t.d();
    if (static_cast<i64>(ranks.size()) != d - 1) fail(Errc::InvalidRanks, "expected d-1 target ranks");
    for (i64 l : ranks)
        if (l < 1) fail(Errc::InvalidRanks, "target ranks must be >= 1");
    if (d == 1) return copy_tt(c, t);
    auto o = orthogonalize_rl_public(c, t);
    return compress_sweep(c, *o, false, 0.0, &ranks);
}

// compression_pass — round_rand.cpp:155-179 (the "Adap-R" second pass): a
// right-to-left sweep over a left-orthogonal TT; per core the QR of H(Y_k)^T,
// a tolerance-truncated SVD of the small triangle, the right-orthogonal core
// (Q V_s)^T kept and U S absorbed into the left neighbour. With R = U_R S V_R^T
// (svd_left of R), R^T = V_R S U_R^T, so U S = R^T U_R and V = U_R: no
// division by singular values.
std::unique_ptr<TTDev> compression_pass(Ctx& c, const TTDev& left, double tau) {
    if (tau < 0) fail(Errc::InvalidArgument, "compression threshold must be >= 0");
    const i64 d = left.d();
    {  // round_rand.cpp:158-163: left-orthogonality defect of cores 0..d-2
        i64 mx = 1;
        for (i64 k = 0; k + 1 < d; ++k) mx = std::max(mx, left.r[k + 1]);
        DBuf G(c, static_cast<std::size_t>(mx * mx));
        for (i64 k = 0; k + 1 < d; ++k) {
            const i64 rows = left.r[k] * left.n[k], cols = left.r[k + 1];
            gemm(c, true, cols, cols, rows, 1.0, left.core(k), rows, left.core(k), rows, 0.0, G.p, cols, false);
            add_diagonal(c, cols, G.p, cols, -1.0);
            if (frob_norm(c, cols, cols, G.p, cols) >= 1e-8)
                fail(Errc::NotLeftOrthogonal, "compression pass requires a left-orthogonal input");
        }
    }
    if (d == 1) return copy_tt(c, left);
    // working copies of the cores (their ranks shrink as the sweep proceeds)
    std::vector<DBuf> cores(static_cast<std::size_t>(d));
    std::vector<i64> r = left.r;
    for (i64 k = 0; k < d; ++k) {
        cores[k] = DBuf(c, static_cast<std::size_t>(left.core_size(k)));
        copy_matrix(c, left.core_size(k), 1, left.core(k), left.core_size(k), cores[k].p, left.core_size(k));
    }
    std::vector<double> s;
    for (i64 k = d - 1; k >= 1; --k) {
        const i64 rl = r[k], nk = left.n[k], rr = r[k + 1], ncols = nk * rr;
        const i64 kk = std::min(ncols, rl);
        // Q R = H(Y_k)^T  (ncols x rl)
        DBuf Ht(c, static_cast<std::size_t>(ncols * rl)), Q(c, static_cast<std::size_t>(ncols * kk)),
            R(c, static_cast<std::size_t>(kk * rl)), U(c, static_cast<std::size_t>(kk * kk));
        transpose(c, rl, ncols, cores[k].p, rl, Ht.p, ncols);
        thin_qr(c, ncols, rl, Ht.p, ncols, Q.p, ncols, R.p, kk);
        // truncated SVD of R^T (orthogonalize.cpp:87-115, tolerance rule)
        svd_left(c, kk, rl, R.p, kk, U.p, kk, s, nullptr);
        const i64 keep = truncation_rank(s, rl, kk, true, tau, 0);
        // core k (horizontal, keep x ncols) = (Q U_R(:, 1:keep))^T
        DBuf P(c, static_cast<std::size_t>(ncols * keep));
        gemm(c, false, ncols, keep, kk, 1.0, Q.p, ncols, U.p, kk, 0.0, P.p, ncols);
        DBuf nk_core(c, static_cast<std::size_t>(keep * ncols));
        transpose(c, ncols, keep, P.p, ncols, nk_core.p, keep);
        cores[k] = std::move(nk_core);
        // core k-1 <- V(core k-1) (U S) with U S = R^T U_R(:, 1:keep)
        DBuf US(c, static_cast<std::size_t>(rl * keep));
        gemm(c, true, rl, keep, kk, 1.0, R.p, kk, U.p, kk, 0.0, US.p, rl);
        const i64 rows_prev = r[k - 1] * left.n[k - 1];
        DBuf prev(c, static_cast<std::size_t>(rows_prev * keep));
        gemm(c, false, rows_prev, keep, rl, 1.0, cores[k - 1].p, rows_prev, US.p, rl, 0.0, prev.p, rows_prev);
        cores[k - 1] = std::move(prev);
        r[k] = keep;
    }
    auto out = std::make_unique<TTDev>(c, left.n, r);
    for (i64 k = 0; k < d; ++k)
        copy_matrix(c, out->core_size(k), 1, cores[k].p, out->core_size(k), out->core(k), out->core_size(k));
    return out;
}

}  // namespace ttr
