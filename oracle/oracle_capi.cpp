// oracle_capi.cpp — extern "C" surface of the CPU oracle for the Python tests
// and bench.py's cpu_baseline leg. TEST INFRASTRUCTURE ONLY.
//
// Status codes follow include/ttround_b200.h: 0 = ok, 1 + Errc index for the
// reference's error kinds (proj/core/include/ttround/types.hpp:15-31), 103 =
// internal. Tensors cross as (d, n[d], r[d+1], concatenated cores in the
// reference layout: core k's vertical unfolding, column-major).
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "ttr_oracle.hpp"

using namespace ttr_oracle;

struct ttro_tt {
    TT tt;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = std::string(errc_name(e.code())) + ": " + e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = std::string("internal: ") + e.what();
        return 103;
    }
}

TT build(std::int64_t d, const std::int64_t* n, const std::int64_t* r, const double* data) {
    std::vector<Core> cores;
    std::int64_t off = 0;
    for (std::int64_t k = 0; k < d; ++k) {
        const std::int64_t cnt = r[k] * n[k] * r[k + 1];
        if (r[k] < 1 || n[k] < 1 || r[k + 1] < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
        cores.emplace_back(r[k], n[k], r[k + 1], std::vector<double>(data + off, data + off + cnt));
        off += cnt;
    }
    return TT(std::move(cores));
}

ttro_tt* wrap(TT t) { return new ttro_tt{std::move(t)}; }

std::vector<Index> vec(const std::int64_t* p, std::int64_t len) { return std::vector<Index>(p, p + len); }
}  // namespace

extern "C" {

const char* ttro_last_error() { return g_err.c_str(); }

int ttro_tt_create(std::int64_t d, const std::int64_t* n, const std::int64_t* r, const double* data, ttro_tt** out) {
    return guard([&] {
        if (d < 1) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
        *out = wrap(build(d, n, r, data));
    });
}
// Per-core shapes (rl[k], n[k], rr[k]); the TT constructor validates the chain
// exactly as tensor.cpp:66-79 does (EmptyCoreList, BoundaryRankNotOne,
// RankChainMismatch).
int ttro_tt_create_chain(std::int64_t d, const std::int64_t* n, const std::int64_t* rl, const std::int64_t* rr,
                         const double* data, ttro_tt** out) {
    return guard([&] {
        std::vector<Core> cores;
        std::int64_t off = 0;
        for (std::int64_t k = 0; k < d; ++k) {
            const std::int64_t cnt = rl[k] * n[k] * rr[k];
            cores.emplace_back(rl[k], n[k], rr[k], std::vector<double>(data + off, data + off + cnt));
            off += cnt;
        }
        *out = wrap(TT(std::move(cores)));
    });
}
void ttro_tt_destroy(ttro_tt* t) { delete t; }

int ttro_tt_shape(const ttro_tt* t, std::int64_t* d, std::int64_t* n, std::int64_t* r, std::int64_t* total) {
    return guard([&] {
        *d = t->tt.order();
        std::int64_t tot = 0;
        if (n) for (std::int64_t k = 0; k < *d; ++k) n[k] = t->tt.core(k).n();
        if (r) for (std::int64_t k = 0; k <= *d; ++k) r[k] = t->tt.rank(k);
        for (std::int64_t k = 0; k < *d; ++k) tot += t->tt.core(k).size();
        if (total) *total = tot;
    });
}
int ttro_tt_order(const ttro_tt* t) { return static_cast<int>(t->tt.order()); }

int ttro_tt_data(const ttro_tt* t, double* out) {
    return guard([&] {
        std::int64_t off = 0;
        for (const auto& c : t->tt.cores()) {
            std::memcpy(out + off, c.data().data(), sizeof(double) * c.data().size());
            off += c.size();
        }
    });
}

int ttro_random_gaussian_tt(std::int64_t d, const std::int64_t* n, const std::int64_t* r, std::uint64_t seed, ttro_tt** out) {
    return guard([&] { *out = wrap(random_gaussian_tt(vec(n, d), vec(r, d + 1), seed)); });
}
int ttro_synthetic(std::int64_t d, std::int64_t n, std::int64_t r, double eps, std::uint64_t seed, ttro_tt** x) {
    return guard([&] { *x = wrap(synthetic_perturbed_tt(d, n, r, eps, seed).x); });
}
int ttro_two_part(std::int64_t d, std::int64_t n, std::int64_t rx, std::int64_t rz, double eps, std::uint64_t seed, ttro_tt** out) {
    return guard([&] { *out = wrap(two_part_tt(d, n, rx, rz, eps, seed)); });
}
int ttro_kernel_sum(std::int64_t d, std::int64_t n, std::int64_t r, std::int64_t terms, double ell, std::uint64_t seed, ttro_tt** out) {
    return guard([&] { *out = wrap(kernel_sum_tt(d, n, r, terms, ell, seed)); });
}
int ttro_formal_sum(const ttro_tt* const* terms, int count, ttro_tt** out) {
    return guard([&] {
        std::vector<TT> ts;
        for (int i = 0; i < count; ++i) ts.push_back(terms[i]->tt);
        *out = wrap(formal_sum(ts));
    });
}
int ttro_scaled(const ttro_tt* t, double alpha, ttro_tt** out) {
    return guard([&] { *out = wrap(scaled(t->tt, alpha)); });
}
int ttro_norm_exact(const ttro_tt* t, double* out) {
    return guard([&] { *out = norm_exact(t->tt); });
}
int ttro_dot(const ttro_tt* a, const ttro_tt* b, double* out) {
    return guard([&] { *out = dot(a->tt, b->tt); });
}
int ttro_relative_error(const ttro_tt* a, const ttro_tt* b, double* out) {
    return guard([&] { *out = relative_error(a->tt, b->tt); });
}
int ttro_entry(const ttro_tt* t, const std::int64_t* idx_one_based, double* out) {
    return guard([&] { *out = t->tt.entry(vec(idx_one_based, t->tt.order())); });
}
int ttro_dense_size(const ttro_tt* t, std::int64_t* size) {
    return guard([&] {
        std::int64_t s = 1;
        for (auto n : t->tt.mode_sizes()) s *= n;
        *size = s;
    });
}
int ttro_contract_to_dense(const ttro_tt* t, std::int64_t max_entries, double* out) {
    return guard([&] {
        auto dn = contract_to_dense(t->tt, max_entries);
        std::memcpy(out, dn.values.data(), sizeof(double) * dn.values.size());
    });
}
int ttro_orthogonalize(const ttro_tt* t, int right_to_left, ttro_tt** out) {
    return guard([&] { *out = wrap(orthogonalize(t->tt, right_to_left ? Direction::RightToLeft : Direction::LeftToRight)); });
}
int ttro_round_det_tol(const ttro_tt* t, double eps, ttro_tt** out) {
    return guard([&] { *out = wrap(round_deterministic(t->tt, eps)); });
}
int ttro_round_det_ranks(const ttro_tt* t, const std::int64_t* ranks, std::int64_t count, ttro_tt** out) {
    return guard([&] { *out = wrap(round_deterministic(t->tt, vec(ranks, count))); });
}
int ttro_round_fixed_krp(const ttro_tt* t, const std::int64_t* ranks, std::int64_t count, std::uint64_t seed, int rng_mode, ttro_tt** out) {
    return guard([&] { *out = wrap(round_fixed_krp(t->tt, vec(ranks, count), seed, static_cast<RngMode>(rng_mode))); });
}
// known_norm: NaN = absent; cap: NULL = absent (else d-1 entries);
// est_out/est_cap: residual estimates in test order; *n_est = count written.
int ttro_round_adaptive_krp(const ttro_tt* t, double tol, double f_init, double f_inc, std::uint64_t seed, int rng_mode,
                            double known_norm, const std::int64_t* cap, ttro_tt** out, double* est_out,
                            std::int64_t est_cap, std::int64_t* n_est, double* tau_out) {
    return guard([&] {
        AdaptiveConfig cfg;
        cfg.tolerance = tol;
        cfg.f_init = f_init;
        cfg.f_inc = f_inc;
        cfg.seed = seed;
        cfg.rng = static_cast<RngMode>(rng_mode);
        if (!std::isnan(known_norm)) cfg.known_norm = known_norm;
        if (cap) cfg.max_rank_cap = vec(cap, t->tt.order() - 1);
        AdaptiveTrace tr;
        *out = wrap(round_adaptive_krp(t->tt, cfg, &tr));
        if (n_est) *n_est = static_cast<std::int64_t>(tr.estimates.size());
        if (est_out)
            for (std::int64_t i = 0; i < std::min<std::int64_t>(est_cap, static_cast<std::int64_t>(tr.estimates.size())); ++i)
                est_out[i] = tr.estimates[static_cast<std::size_t>(i)];
        if (tau_out) *tau_out = tr.tau;
    });
}
int ttro_round_rand_orth_tt(const ttro_tt* t, const std::int64_t* ranks, std::int64_t count, std::uint64_t seed,
                            int rng_mode, ttro_tt** out) {
    return guard([&] { *out = wrap(round_rand_orth_tt(t->tt, vec(ranks, count), seed, static_cast<RngMode>(rng_mode))); });
}

int ttro_tt_partial_contractions(const ttro_tt* x, const ttro_tt* r, double* out) {
    return guard([&] {
        auto w = tt_partial_contractions_rl(x->tt, r->tt);
        std::size_t o = 0;
        for (const auto& m : w) {
            std::copy(m.a.begin(), m.a.end(), out + o);
            o += m.a.size();
        }
    });
}

int ttro_round_sum_adaptive_krp(const ttro_tt* const* terms, int count, double eps, double f_inc, std::uint64_t seed,
                                int rng_mode, ttro_tt** out) {
    return guard([&] {
        std::vector<TT> ts;
        for (int i = 0; i < count; ++i) ts.push_back(terms[i]->tt);
        *out = wrap(round_sum_adaptive_krp(ts, eps, f_inc, seed, static_cast<RngMode>(rng_mode)));
    });
}

// TT-GMRES on the cookie problem (solver.cpp:241-363): config as plain values,
// histories into caller buffers of capacity max_iterations.
int ttro_gmres_cookie(std::int64_t p, std::int64_t grid, std::int64_t samples, double rho_min, double rho_max,
                      double rel_tol, std::int64_t max_it, int strategy, double rounding_tol, std::uint64_t seed,
                      int track_true, int precond, int rng_mode, std::int64_t* iterations, int* converged,
                      double* residual_hist, double* true_hist, std::int64_t* rank_hist, ttro_tt** solution) {
    return guard([&] {
        CookieProblem prob = build_cookie_problem(p, grid, samples, rho_min, rho_max);
        GmresConfig cfg;
        cfg.rel_tolerance = rel_tol;
        cfg.max_iterations = max_it;
        cfg.strategy = static_cast<GmresStrategy>(strategy);
        cfg.rounding_tolerance = rounding_tol;
        cfg.seed = seed;
        cfg.track_true_residual = track_true != 0;
        cfg.mean_field_preconditioner = precond != 0;
        cfg.rng = static_cast<RngMode>(rng_mode);
        GmresResult r = tt_gmres(prob.op, prob.rhs, cfg);
        *iterations = r.iterations;
        *converged = r.converged ? 1 : 0;
        for (std::size_t i = 0; i < r.residual_history.size(); ++i) residual_hist[i] = r.residual_history[i];
        for (std::size_t i = 0; i < r.true_residual_history.size(); ++i) true_hist[i] = r.true_residual_history[i];
        for (std::size_t i = 0; i < r.max_rank_history.size(); ++i) rank_hist[i] = r.max_rank_history[i];
        *solution = wrap(std::move(r.solution));
    });
}

// The cookie operator's factors A_{i,k} (column-major, term-major then mode)
// and the right-hand side (build_cookie_problem, solver.cpp:81-135).
int ttro_cookie_problem(std::int64_t p, std::int64_t grid, std::int64_t samples, double rho_min, double rho_max,
                        double* factors, ttro_tt** rhs) {
    return guard([&] {
        CookieProblem prob = build_cookie_problem(p, grid, samples, rho_min, rho_max);
        std::int64_t off = 0;
        for (const auto& term : prob.op.terms)
            for (const auto& a : term) {
                std::memcpy(factors + off, a.data(), sizeof(double) * a.a.size());
                off += static_cast<std::int64_t>(a.a.size());
            }
        *rhs = wrap(std::move(prob.rhs));
    });
}

// apply_operator of an explicit operator (factors as above, nterms x d) to t:
// the nterms result terms.
int ttro_apply_operator(std::int64_t nterms, const double* factors, const ttro_tt* t, ttro_tt** out) {
    return guard([&] {
        const auto modes = t->tt.mode_sizes();
        std::vector<std::vector<Matrix>> terms;
        std::int64_t off = 0;
        for (std::int64_t i = 0; i < nterms; ++i) {
            std::vector<Matrix> term;
            for (Index n : modes) {
                Matrix a(n, n);
                std::memcpy(a.data(), factors + off, sizeof(double) * n * n);
                off += n * n;
                term.push_back(std::move(a));
            }
            terms.push_back(std::move(term));
        }
        auto res = apply_operator(KronOp::of(std::move(terms)), t->tt);
        for (std::size_t i = 0; i < res.size(); ++i) out[i] = wrap(std::move(res[i]));
    });
}

int ttro_compression_pass(const ttro_tt* t, double tau, ttro_tt** out) {
    return guard([&] { *out = wrap(compression_pass(t->tt, tau)); });
}
int ttro_estimate_norm_krp(const ttro_tt* t, std::int64_t width, std::uint64_t seed, int rng_mode, double* out) {
    return guard([&] { *out = estimate_norm_krp(t->tt, width, seed, static_cast<RngMode>(rng_mode)); });
}
// Factors Omega_start..Omega_d (n_k x cols each, column-major, concatenated).
int ttro_draw_factors(const ttro_tt* t, std::int64_t start_mode, std::int64_t cols, std::uint64_t seed, int rng_mode,
                      std::int64_t col0, double* out) {
    return guard([&] {
        FactorRng rng(static_cast<RngMode>(rng_mode), seed);
        auto f = draw_gaussian_factors(t->tt, start_mode, cols, rng, col0);
        std::int64_t off = 0;
        for (const auto& m : f.factors) {
            std::memcpy(out + off, m.data(), sizeof(double) * m.a.size());
            off += static_cast<std::int64_t>(m.a.size());
        }
    });
}
// W_start..W_d (r_{k-1} x cols, concatenated) for given factors.
int ttro_krp_contractions(const ttro_tt* t, std::int64_t start_mode, std::int64_t cols, const double* factors, double* out) {
    return guard([&] {
        FactorSet f;
        f.start_mode = start_mode;
        std::int64_t off = 0;
        for (std::int64_t k = start_mode; k <= t->tt.order(); ++k) {
            const std::int64_t n = t->tt.core(k - 1).n();
            Matrix m(n, cols);
            std::memcpy(m.data(), factors + off, sizeof(double) * static_cast<std::size_t>(n * cols));
            off += n * cols;
            f.factors.push_back(std::move(m));
        }
        auto w = krp_partial_contractions_rl(t->tt, f);
        off = 0;
        for (const auto& m : w.w) {
            std::memcpy(out + off, m.data(), sizeof(double) * m.a.size());
            off += static_cast<std::int64_t>(m.a.size());
        }
    });
}
// generate_residual_sketch (round_rand.cpp:80-94) after an initial contraction of
// width w0 from mode 2 (the adaptive driver's sequence): S (rows x b) and the
// widths of W_2..W_d afterwards.
int ttro_residual_sketch(const ttro_tt* t, std::int64_t w0, std::uint64_t seed, int rng_mode, std::int64_t rows,
                         std::int64_t zc, const double* z, std::int64_t qc, const double* q, std::int64_t k,
                         std::int64_t b, double* s_out, std::int64_t* widths) {
    return guard([&] {
        FactorRng rng(static_cast<RngMode>(rng_mode), seed);
        auto f = draw_gaussian_factors(t->tt, 2, w0, rng);
        auto w = krp_partial_contractions_rl(t->tt, f);
        Matrix zm(rows, zc), qm(rows, qc);
        std::memcpy(zm.data(), z, sizeof(double) * static_cast<std::size_t>(rows * zc));
        if (qc) std::memcpy(qm.data(), q, sizeof(double) * static_cast<std::size_t>(rows * qc));
        Matrix s = generate_residual_sketch(t->tt, zm, qm, w, k, b, rng);
        std::memcpy(s_out, s.data(), sizeof(double) * s.a.size());
        for (std::size_t i = 0; i < w.w.size(); ++i) widths[i] = w.w[i].cols;
    });
}
int ttro_residual_norm_estimate(std::int64_t rows, std::int64_t cols, const double* s, std::int64_t block, double* out) {
    return guard([&] {
        Matrix m(rows, cols);
        if (rows > 0 && cols > 0) std::memcpy(m.data(), s, sizeof(double) * static_cast<std::size_t>(rows * cols));
        *out = residual_norm_estimate(m, block);
    });
}
int ttro_gaussian_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
    return guard([&] {
        auto m = gaussian_matrix(rows, cols, seed);
        std::memcpy(out, m.data(), sizeof(double) * m.a.size());
    });
}
int ttro_derive_seed(std::uint64_t seed, std::uint64_t tag, std::uint64_t* out) {
    *out = derive_seed(seed, tag);
    return 0;
}
int ttro_philox_factor(std::uint64_t seed, std::int64_t mode, std::int64_t rows, std::int64_t cols, std::int64_t col0, double* out) {
    return guard([&] {
        auto m = philox_factor(seed, mode, rows, cols, col0);
        std::memcpy(out, m.data(), sizeof(double) * m.a.size());
    });
}
int ttro_thin_qr(std::int64_t rows, std::int64_t cols, const double* a, double* q, double* r) {
    return guard([&] {
        Matrix m(rows, cols);
        std::memcpy(m.data(), a, sizeof(double) * static_cast<std::size_t>(rows * cols));
        auto f = linalg::thin_qr(m);
        if (q) std::memcpy(q, f.q.data(), sizeof(double) * f.q.a.size());
        if (r) std::memcpy(r, f.r.data(), sizeof(double) * f.r.a.size());
    });
}
int ttro_truncated_svd(std::int64_t rows, std::int64_t cols, const double* a, int tol_rule, double tau, std::int64_t l,
                       std::int64_t* rank, double* u, double* s, double* v) {
    return guard([&] {
        Matrix m(rows, cols);
        std::memcpy(m.data(), a, sizeof(double) * static_cast<std::size_t>(rows * cols));
        auto t = tol_rule ? truncated_svd_tol(m, tau) : truncated_svd_rank(m, l);
        *rank = t.rank;
        if (u) std::memcpy(u, t.u.data(), sizeof(double) * t.u.a.size());
        if (s) std::memcpy(s, t.s.data(), sizeof(double) * t.s.size());
        if (v) std::memcpy(v, t.v.data(), sizeof(double) * t.v.a.size());
    });
}
int ttro_set_backend(int backend, int threads) { return guard([&] { linalg::set_backend(backend, threads); }); }
int ttro_backend() { return linalg::backend(); }
int ttro_blas_available() { return linalg::blas_available() ? 1 : 0; }
int ttro_random_philox_tt(std::int64_t d, const std::int64_t* n, const std::int64_t* r, std::uint64_t seed,
                          ttro_tt** out) {
    return guard([&] { *out = wrap(random_philox_tt(vec(n, d), vec(r, d + 1), seed)); });
}
void ttro_flops_reset() { flops::reset(); }
void ttro_flops_get(std::uint64_t* out5) {
    const auto& c = flops::counters();
    out5[0] = c.gemm;
    out5[1] = c.qr;
    out5[2] = c.svd;
    out5[3] = c.sketch;
    out5[4] = c.rng;
}

// CPU-baseline timing helpers (bench.py): wall clock around the call only,
// as tools/ttround_main.cpp:156-160 does.
int ttro_time_round_fixed_krp(const ttro_tt* t, const std::int64_t* ranks, std::int64_t count, std::uint64_t seed,
                              int rng_mode, double* seconds, std::uint64_t* flops_total) {
    return guard([&] {
        flops::reset();
        const auto t0 = std::chrono::steady_clock::now();
        TT y = round_fixed_krp(t->tt, vec(ranks, count), seed, static_cast<RngMode>(rng_mode));
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *flops_total = flops::counters().total();
    });
}
}  // extern "C"
