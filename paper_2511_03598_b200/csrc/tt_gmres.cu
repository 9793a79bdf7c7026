// tt_gmres.cu — the reference's TT-GMRES "cookie" harness on the device
// (proj/core/src/solver.cpp, include/ttround/solver.hpp): the
// caller that drives Sum+Round. The Kronecker-sum operator lives on the device
// (one n_k x n_k factor per term and mode, stored transposed), operator
// application is one strided-batch DMMA GEMM per non-identity factor and core
// (out_b = X_b A^T over the r_k slabs), every Sum+Round is one of the device
// roundings (TT-SVD, Rand-Orth TT + compression pass, adaptive KRP sum +
// compression pass), and only the Arnoldi scalars (dots, norms, the Givens
// least-squares) live on the host, as in the reference.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>

#include "common.cuh"
#include "rng_host.h"
#include "tt_gmres.h"

namespace ttr {
namespace {

// solver.cpp:41-66 — 5-point flux-form finite differences of -div(chi grad u)
// on the grid x grid interior of the unit square (chi at edge midpoints);
// column-major grid^2 x grid^2
std::vector<double> fd_diffusion_matrix(i64 grid, const std::function<double(double, double)>& chi) {
    const i64 n = grid * grid;
    const double h = 1.0 / static_cast<double>(grid + 1);
    std::vector<double> a(static_cast<std::size_t>(n * n), 0.0);
    const i64 dx[4] = {1, -1, 0, 0}, dy[4] = {0, 0, 1, -1};
    for (i64 iy = 0; iy < grid; ++iy)
        for (i64 ix = 0; ix < grid; ++ix) {
            const double x = (ix + 1) * h, y = (iy + 1) * h;
            const i64 row = iy * grid + ix;
            for (int e = 0; e < 4; ++e) {
                const double c = chi(x + 0.5 * h * dx[e], y + 0.5 * h * dy[e]) / (h * h);
                if (c == 0.0) continue;
                a[static_cast<std::size_t>(row + row * n)] += c;
                const i64 jx = ix + dx[e], jy = iy + dy[e];
                if (jx >= 0 && jx < grid && jy >= 0 && jy < grid) a[static_cast<std::size_t>(row + (jy * grid + jx) * n)] -= c;
            }
        }
    return a;
}

// Eigen::PartialPivLU of the mean-field matrix, inverted once on the host
// (setup, O(n^3) with n = grid^2): the mode-1 solve becomes one GEMM.
std::vector<double> lu_inverse(std::vector<double> a, i64 n) {
    std::vector<i64> perm(static_cast<std::size_t>(n));
    for (i64 i = 0; i < n; ++i) perm[static_cast<std::size_t>(i)] = i;
    auto at = [&](i64 i, i64 j) -> double& { return a[static_cast<std::size_t>(i + j * n)]; };
    for (i64 k = 0; k < n; ++k) {
        i64 p = k;
        for (i64 i = k + 1; i < n; ++i)
            if (std::fabs(at(i, k)) > std::fabs(at(p, k))) p = i;
        if (at(p, k) == 0.0) fail(Errc::Breakdown, "mean-field preconditioner is singular");
        if (p != k) {
            for (i64 j = 0; j < n; ++j) std::swap(at(k, j), at(p, j));
            std::swap(perm[static_cast<std::size_t>(k)], perm[static_cast<std::size_t>(p)]);
        }
        const double piv = at(k, k);
        for (i64 i = k + 1; i < n; ++i) at(i, k) /= piv;
        for (i64 j = k + 1; j < n; ++j) {
            const double u = at(k, j);
            if (u == 0.0) continue;
            for (i64 i = k + 1; i < n; ++i) at(i, j) -= at(i, k) * u;
        }
    }
    std::vector<double> inv(static_cast<std::size_t>(n * n), 0.0);
    std::vector<double> x(static_cast<std::size_t>(n));
    for (i64 c = 0; c < n; ++c) {  // column c of A^{-1}: solve L U x = P e_c
        for (i64 i = 0; i < n; ++i) x[static_cast<std::size_t>(i)] = perm[static_cast<std::size_t>(i)] == c ? 1.0 : 0.0;
        for (i64 i = 0; i < n; ++i)
            for (i64 k = 0; k < i; ++k) x[static_cast<std::size_t>(i)] -= at(i, k) * x[static_cast<std::size_t>(k)];
        for (i64 i = n - 1; i >= 0; --i) {
            for (i64 k = i + 1; k < n; ++k) x[static_cast<std::size_t>(i)] -= at(i, k) * x[static_cast<std::size_t>(k)];
            x[static_cast<std::size_t>(i)] /= at(i, i);
        }
        std::memcpy(inv.data() + c * n, x.data(), sizeof(double) * static_cast<std::size_t>(n));
    }
    return inv;
}

std::unique_ptr<TTDev> scaled_copy(Ctx& c, const TTDev& t, double alpha) {
    auto out = copy_tt(c, t);
    scale_tt(c, *out, alpha);
    return out;
}

double left_orthogonal_norm(Ctx& c, const TTDev& t) {  // solver.cpp:157-159
    const i64 k = t.d() - 1;
    return frob_norm(c, t.core_size(k), 1, t.core(k), t.core_size(k));
}

// solver.cpp:161-212
class SumRounder {
public:
    SumRounder(Ctx& c, int strategy, double delta, std::uint64_t seed, int rng)
        : c_(c), s_(strategy), delta_(delta), seed_(seed), rng_(rng) {}
    std::unique_ptr<TTDev> round(const std::vector<const TTDev*>& terms) {
        const auto t0 = std::chrono::steady_clock::now();
        auto out = impl(terms);
        TTR_CUDA(cudaStreamSynchronize(c_.stream));
        seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return out;
    }
    double seconds() const { return seconds_; }

private:
    std::unique_ptr<TTDev> impl(const std::vector<const TTDev*>& terms) {
        const std::uint64_t seed = derive_seed(seed_, counter_++);
        switch (s_) {
            case TTR_GMRES_DETERMINISTIC:
                return round_deterministic_tol(c_, *formal_sum(c_, terms), delta_);
            case TTR_GMRES_RAND_ORTH_TT: {
                auto f = formal_sum(c_, terms);
                if (f->d() == 1) return f;
                // sketch at the formal-sum ranks: lossless projection, the
                // compression pass owns the truncation
                std::vector<i64> targets(f->r.begin() + 1, f->r.end() - 1);
                auto y = round_rand_orth_tt(c_, *f, targets, seed, rng_);
                const double tau = delta_ * left_orthogonal_norm(c_, *y) / std::sqrt(static_cast<double>(y->d() - 1));
                return compression_pass(c_, *y, tau);
            }
            case TTR_GMRES_ADAPTIVE_KRP_SUM: {
                auto y = round_sum_adaptive_krp(c_, terms, delta_, 0.05, seed, rng_);
                if (y->d() == 1) return y;
                const double nrm = left_orthogonal_norm(c_, *y);
                if (nrm == 0.0) return y;  // the cancellation guard's zero tensor
                return compression_pass(c_, *y, delta_ * nrm / std::sqrt(static_cast<double>(y->d() - 1)));
            }
        }
        fail(Errc::InvalidArgument, "unknown rounding strategy");
    }
    Ctx& c_;
    int s_;
    double delta_;
    std::uint64_t seed_;
    int rng_;
    std::uint64_t counter_ = 0;
    double seconds_ = 0.0;
};

}  // namespace

KronOpDev::KronOpDev(Ctx& c, i64 nterms_, const std::vector<i64>& n_, const double* factors)
    : n(n_), nterms(nterms_) {  // KroneckerSumOperator::of, solver.cpp:16-30
    if (nterms < 1) fail(Errc::InvalidArgument, "operator needs at least one term");
    if (n.empty()) fail(Errc::InvalidArgument, "operator term needs at least one factor");
    for (i64 k : n)
        if (k < 1) fail(Errc::ModeSizeMismatch, "operator factors must be square and consistent");
    const i64 d = static_cast<i64>(n.size());
    i64 off = 0;
    host.resize(static_cast<std::size_t>(nterms));
    At.resize(static_cast<std::size_t>(nterms));
    identity.resize(static_cast<std::size_t>(nterms));
    for (i64 i = 0; i < nterms; ++i) {
        for (i64 k = 0; k < d; ++k) {
            const i64 m = n[static_cast<std::size_t>(k)];
            std::vector<double> a(factors + off, factors + off + m * m);
            off += m * m;
            bool eye = true;
            for (i64 q = 0; q < m && eye; ++q)
                for (i64 p = 0; p < m; ++p)
                    if (a[static_cast<std::size_t>(p + q * m)] != (p == q ? 1.0 : 0.0)) {
                        eye = false;
                        break;
                    }
            std::vector<double> at(static_cast<std::size_t>(m * m));
            for (i64 q = 0; q < m; ++q)
                for (i64 p = 0; p < m; ++p) at[static_cast<std::size_t>(q + p * m)] = a[static_cast<std::size_t>(p + q * m)];
            DBuf dbuf(c, static_cast<std::size_t>(m * m));
            TTR_CUDA(cudaMemcpyAsync(dbuf.p, at.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, c.stream));
            TTR_CUDA(cudaStreamSynchronize(c.stream));  // host staging lifetime
            host[static_cast<std::size_t>(i)].push_back(std::move(a));
            At[static_cast<std::size_t>(i)].push_back(std::move(dbuf));
            identity[static_cast<std::size_t>(i)].push_back(eye);
        }
    }
}

std::unique_ptr<KronOpDev> cookie_problem(Ctx& c, i64 p, i64 grid, i64 samples, double rho_min, double rho_max,
                                          std::unique_ptr<TTDev>* rhs) {  // solver.cpp:81-135
    if (grid < 8) fail(Errc::InvalidGrid, "grid size must be >= 8");
    if (p < 0) fail(Errc::InvalidGrid, "parameter mode count must be >= 0");
    if (p > 0 && samples < 1) fail(Errc::InvalidGrid, "need at least one parameter sample");
    if (rho_max < rho_min) fail(Errc::InvalidGrid, "empty parameter range");
    const i64 d = p + 1;
    std::vector<i64> modes(static_cast<std::size_t>(d), samples);
    modes[0] = grid * grid;
    const i64 cells = p > 0 ? static_cast<i64>(std::ceil(std::sqrt(static_cast<double>(p)))) : 1;
    const double radius = 0.35 / static_cast<double>(cells);
    std::vector<double> rho(static_cast<std::size_t>(std::max<i64>(samples, 0)));
    for (i64 i = 0; i < samples; ++i)
        rho[static_cast<std::size_t>(i)] =
            samples == 1 ? rho_min
                         : rho_min + (rho_max - rho_min) * static_cast<double>(i) / static_cast<double>(samples - 1);
    std::vector<double> factors;
    auto push_eye = [&](i64 m) {
        for (i64 q = 0; q < m; ++q)
            for (i64 r = 0; r < m; ++r) factors.push_back(r == q ? 1.0 : 0.0);
    };
    auto push = [&](const std::vector<double>& a) { factors.insert(factors.end(), a.begin(), a.end()); };
    push(fd_diffusion_matrix(grid, [](double, double) { return 1.0; }));
    for (i64 k = 1; k < d; ++k) push_eye(modes[static_cast<std::size_t>(k)]);
    for (i64 i = 0; i < p; ++i) {
        const double cx = (i % cells + 0.5) / static_cast<double>(cells), cy = (i / cells + 0.5) / static_cast<double>(cells);
        push(fd_diffusion_matrix(grid, [cx, cy, radius](double x, double y) {
            const double ddx = x - cx, ddy = y - cy;
            return ddx * ddx + ddy * ddy <= radius * radius ? 1.0 : 0.0;
        }));
        for (i64 k = 1; k < d; ++k) {
            if (k == i + 1) {
                for (i64 q = 0; q < samples; ++q)
                    for (i64 r = 0; r < samples; ++r) factors.push_back(r == q ? rho[static_cast<std::size_t>(q)] : 0.0);
            } else {
                push_eye(modes[static_cast<std::size_t>(k)]);
            }
        }
    }
    auto op = std::make_unique<KronOpDev>(c, p + 1, modes, factors.data());
    // right-hand side: the rank-1 TT of ones (solver.cpp:68-77)
    std::vector<i64> r(static_cast<std::size_t>(d + 1), 1);
    *rhs = std::make_unique<TTDev>(c, modes, r);
    for (i64 k = 0; k < d; ++k) fill(c, (*rhs)->core(k), static_cast<std::size_t>((*rhs)->core_size(k)), 1.0);
    return op;
}

std::vector<std::unique_ptr<TTDev>> apply_operator(Ctx& c, const KronOpDev& op, const TTDev& x) {  // solver.cpp:137-151
    if (op.n != x.n) fail(Errc::ModeSizeMismatch, "operator and tensor mode sizes differ");
    std::vector<std::unique_ptr<TTDev>> out;
    const i64 d = x.d();
    for (i64 i = 0; i < op.nterms; ++i) {
        auto t = std::make_unique<TTDev>(c, x.n, x.r);
        for (i64 k = 0; k < d; ++k) {
            const i64 rl = x.r[k], nk = x.n[k], rr = x.r[k + 1];
            if (op.identity[static_cast<std::size_t>(i)][static_cast<std::size_t>(k)]) {
                TTR_CUDA(cudaMemcpyAsync(t->core(k), x.core(k), sizeof(double) * rl * nk * rr, cudaMemcpyDeviceToDevice,
                                         c.stream));
                continue;
            }
            // out(:, :, b) = X(:, :, b) A^T for every slab b (detail::contract_mode)
            gemm_batched(c, false, rl, nk, nk, 1.0, x.core(k), rl, rl * nk,
                         op.At[static_cast<std::size_t>(i)][static_cast<std::size_t>(k)].p, nk, 0, 0.0, t->core(k), rl,
                         rl * nk, rr);
        }
        out.push_back(std::move(t));
    }
    return out;
}

GmresResultDev tt_gmres(Ctx& c, const KronOpDev& op, const TTDev& rhs, const ttr_gmres_cfg& cfg) {  // solver.cpp:241-363
    if (!(cfg.rel_tolerance > 0.0)) fail(Errc::InvalidArgument, "solver tolerance must be > 0");
    if (op.n != rhs.n) fail(Errc::ModeSizeMismatch, "operator and rhs mode sizes differ");
    if (cfg.max_iterations < 1) fail(Errc::InvalidArgument, "max_iterations must be >= 1");
    const double delta = cfg.rounding_tolerance > 0.0 ? cfg.rounding_tolerance : 0.1 * cfg.rel_tolerance;
    const i64 m = cfg.max_iterations;
    SumRounder rounder(c, cfg.strategy, delta, cfg.seed, cfg.rng_mode);
    // right preconditioning with the mean-field spatial operator (solver.cpp:218-237):
    // M = sum_i (prod_{k>=2} mean diag A_{i,k}) A_{i,1}, inverted once
    DBuf minv;
    const i64 n1 = op.n[0];
    if (cfg.mean_field_preconditioner) {
        std::vector<double> mf(static_cast<std::size_t>(n1 * n1), 0.0);
        for (i64 i = 0; i < op.nterms; ++i) {
            double w = 1.0;
            for (std::size_t k = 1; k < op.n.size(); ++k) {
                const auto& a = op.host[static_cast<std::size_t>(i)][k];
                double s = 0.0;
                for (i64 q = 0; q < op.n[k]; ++q) s += a[static_cast<std::size_t>(q + q * op.n[k])];
                w *= s / static_cast<double>(op.n[k]);
            }
            const auto& a0 = op.host[static_cast<std::size_t>(i)][0];
            for (std::size_t e = 0; e < mf.size(); ++e) mf[e] += w * a0[e];
        }
        auto inv = lu_inverse(std::move(mf), n1);
        minv = DBuf(c, static_cast<std::size_t>(n1 * n1));
        TTR_CUDA(cudaMemcpyAsync(minv.p, inv.data(), sizeof(double) * n1 * n1, cudaMemcpyHostToDevice, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
    }
    auto solve_mode1 = [&](const TTDev& x) {  // the mode-1 solve of every core-1 column (one GEMM)
        auto y = copy_tt(c, x);
        const i64 r1 = x.r[1];
        gemm(c, false, n1, r1, n1, 1.0, minv.p, n1, x.core(0), n1, 0.0, y->core(0), n1);
        return y;
    };
    GmresResultDev res;
    {
        std::vector<i64> r1(rhs.n.size() + 1, 1);
        res.solution = std::make_unique<TTDev>(c, rhs.n, r1);
        for (i64 k = 0; k < res.solution->d(); ++k)
            fill(c, res.solution->core(k), static_cast<std::size_t>(res.solution->core_size(k)), 0.0);
    }
    const double normb = norm_exact(c, rhs);
    if (normb == 0.0) {
        res.converged = true;
        return res;
    }
    std::vector<std::unique_ptr<TTDev>> basis;
    basis.push_back(scaled_copy(c, rhs, 1.0 / normb));
    std::vector<double> hess(static_cast<std::size_t>((m + 1) * m), 0.0);
    auto H = [&](i64 i, i64 j) -> double& { return hess[static_cast<std::size_t>(i + j * (m + 1))]; };
    std::vector<double> g(static_cast<std::size_t>(m + 1), 0.0), cs(static_cast<std::size_t>(m), 0.0),
        sn(static_cast<std::size_t>(m), 0.0);
    g[0] = normb;
    auto solve_iterate = [&](i64 j) {
        std::vector<double> y(g.begin(), g.begin() + j + 1);
        for (i64 i = j; i >= 0; --i) {
            for (i64 l = i + 1; l <= j; ++l) y[static_cast<std::size_t>(i)] -= H(i, l) * y[static_cast<std::size_t>(l)];
            y[static_cast<std::size_t>(i)] /= H(i, i);
        }
        std::vector<std::unique_ptr<TTDev>> combo;
        std::vector<const TTDev*> ptrs;
        for (i64 i = 0; i <= j; ++i) {
            combo.push_back(scaled_copy(c, *basis[static_cast<std::size_t>(i)], y[static_cast<std::size_t>(i)]));
            ptrs.push_back(combo.back().get());
        }
        auto x = rounder.round(ptrs);
        return cfg.mean_field_preconditioner ? solve_mode1(*x) : std::move(x);
    };
    auto true_residual = [&](const TTDev& x) {
        auto ax = apply_operator(c, op, x);
        std::vector<const TTDev*> diff{&rhs};
        for (auto& t : ax) {
            scale_tt(c, *t, -1.0);
            diff.push_back(t.get());
        }
        return norm_exact(c, *formal_sum(c, diff)) / normb;
    };
    for (i64 j = 0; j < m; ++j) {
        const TTDev& v = *basis[static_cast<std::size_t>(j)];
        std::vector<std::unique_ptr<TTDev>> aw;
        if (cfg.mean_field_preconditioner) aw = apply_operator(c, op, *solve_mode1(v));
        else aw = apply_operator(c, op, v);
        std::vector<const TTDev*> awp;
        for (auto& t : aw) awp.push_back(t.get());
        auto w = rounder.round(awp);
        aw.clear();
        for (i64 i = 0; i <= j; ++i) {  // modified Gram-Schmidt, Sum+Round after every subtraction
            const double hij = dot(c, *w, *basis[static_cast<std::size_t>(i)]);
            H(i, j) = hij;
            auto sb = scaled_copy(c, *basis[static_cast<std::size_t>(i)], -hij);
            w = rounder.round({w.get(), sb.get()});
        }
        const double hj1 = norm_exact(c, *w);
        H(j + 1, j) = hj1;
        for (i64 i = 0; i < j; ++i) {
            const double t = cs[static_cast<std::size_t>(i)] * H(i, j) + sn[static_cast<std::size_t>(i)] * H(i + 1, j);
            H(i + 1, j) = -sn[static_cast<std::size_t>(i)] * H(i, j) + cs[static_cast<std::size_t>(i)] * H(i + 1, j);
            H(i, j) = t;
        }
        const double denom = std::hypot(H(j, j), H(j + 1, j));
        if (denom == 0.0) {
            cs[static_cast<std::size_t>(j)] = 1.0;
            sn[static_cast<std::size_t>(j)] = 0.0;
        } else {
            cs[static_cast<std::size_t>(j)] = H(j, j) / denom;
            sn[static_cast<std::size_t>(j)] = H(j + 1, j) / denom;
        }
        H(j, j) = denom;
        H(j + 1, j) = 0.0;
        g[static_cast<std::size_t>(j + 1)] = -sn[static_cast<std::size_t>(j)] * g[static_cast<std::size_t>(j)];
        g[static_cast<std::size_t>(j)] = cs[static_cast<std::size_t>(j)] * g[static_cast<std::size_t>(j)];
        const double estimate = std::fabs(g[static_cast<std::size_t>(j + 1)]) / normb;
        res.residual_history.push_back(estimate);
        res.max_rank_history.push_back(w->max_rank());
        res.rounding_seconds_history.push_back(rounder.seconds());
        res.iterations = j + 1;
        const bool stagnated = hj1 <= 1e-14 * normb;
        const bool stopping = estimate <= cfg.rel_tolerance || stagnated || j + 1 == m;
        double true_res = estimate;
        if (cfg.track_true_residual || stopping) {
            auto x = solve_iterate(j);
            true_res = true_residual(*x);
            res.solution = std::move(x);
        }
        if (cfg.track_true_residual) res.true_residual_history.push_back(true_res);
        if (estimate <= cfg.rel_tolerance) {
            res.converged = true;
            break;
        }
        if (stagnated) {
            if (true_res <= cfg.rel_tolerance) {
                res.converged = true;
                break;
            }
            fail(Errc::Breakdown, "Arnoldi vector norm vanished before convergence");
        }
        scale_tt(c, *w, 1.0 / hj1);
        basis.push_back(std::move(w));
    }
    res.rounding_seconds = rounder.seconds();
    return res;
}

}  // namespace ttr
