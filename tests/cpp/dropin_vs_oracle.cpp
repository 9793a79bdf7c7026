// The drop-in C++ layer (include/ttround_b200/ttround.hpp) against the CPU
// oracle, entry point by entry point: every function of the reference's
// tensor / sketch / rounding headers that the layer mirrors is called on the
// device and compared with the oracle's restatement of the reference on the
// same input and the same (reference xoshiro) stream. TEST INFRASTRUCTURE:
// links the oracle (oracle/_build/libttr_oracle.so) only as the checker.
// Prints one "dropin ok" line; a non-zero exit code names the failed check.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../oracle/ttr_oracle.hpp"
#include "ttround_b200/ttround.hpp"

namespace O = ttr_oracle;
namespace T = ttround;

static int g_fail = 0;
#define EXPECT(cond, what)                                          \
    do {                                                            \
        if (!(cond)) {                                              \
            std::printf("FAIL %s (line %d)\n", what, __LINE__);     \
            if (!g_fail) g_fail = __LINE__;                         \
        }                                                           \
    } while (0)

static T::TTTensor to_device(const O::TT& x) {
    std::vector<T::Core> cores;
    for (const auto& c : x.cores()) cores.emplace_back(c.r_left(), c.n(), c.r_right(), c.data());
    return T::TTTensor(cores);
}

static O::TT to_oracle(const T::TTTensor& y) {
    std::vector<O::Core> cores;
    for (T::Index k = 0; k < y.order(); ++k) {
        T::Core c = y.core(k);
        cores.emplace_back(c.r_left(), c.n(), c.r_right(), c.data());
    }
    return O::TT(std::move(cores));
}

static double max_rel(const T::Matrix& a, const O::Matrix& b) {
    if (a.rows() != b.rows || a.cols() != b.cols) return 1e300;
    double diff = 0, nrm = 0;
    for (std::size_t i = 0; i < a.a.size(); ++i) {
        diff = std::max(diff, std::abs(a.a[i] - b.a[i]));
        nrm = std::max(nrm, std::abs(b.a[i]));
    }
    return diff / (1.0 + nrm);
}

static bool bitwise(const T::Matrix& a, const O::Matrix& b) {
    return a.rows() == b.rows && a.cols() == b.cols && a.a == b.a;
}

template <typename F>
static T::Errc errc_of(F&& f) {
    try {
        f();
    } catch (const T::Error& e) {
        return e.code();
    }
    return T::Errc::DeviceFailure;  // "no error" sentinel for the checks below
}

int main() {
    try {
        const O::TT xo = O::two_part_tt(6, 12, 5, 9, 1e-3, 4242);
        const T::TTTensor x = to_device(xo);

        // Core / TTTensor(std::vector<Core>) round trip, tensor.hpp:17-63
        for (T::Index k = 0; k < x.order(); ++k) EXPECT(x.core(k).data() == xo.core(k).data(), "core round trip");
        EXPECT(x.ranks() == xo.ranks(), "ranks");

        // random_gaussian_tt (reference stream, bitwise) and dot, tensor.hpp:111,119
        const std::vector<T::Index> modes{7, 5, 6, 4}, ranks{1, 3, 4, 2, 1};
        const T::TTTensor g = T::random_gaussian_tt(modes, ranks, 99);
        const O::TT go = O::random_gaussian_tt(modes, ranks, 99);
        for (T::Index k = 0; k < 4; ++k) EXPECT(g.core(k).data() == go.core(k).data(), "random_gaussian_tt bitwise");
        const O::TT ho = O::random_gaussian_tt(modes, {1, 2, 5, 3, 1}, 7);
        const double dg = T::dot(g, to_device(ho)), dr = O::dot(go, ho);
        EXPECT(std::abs(dg - dr) <= 1e-12 * (std::abs(dr) + O::norm_exact(go) * O::norm_exact(ho)), "dot");
        EXPECT(std::abs(T::norm_exact(x) - O::norm_exact(xo)) <= 1e-12 * O::norm_exact(xo), "norm_exact");
        const O::TT so = O::formal_sum({xo, O::scaled(xo, -0.5)});
        const T::TTTensor sd = T::formal_sum({x, T::scaled(x, -0.5)});
        EXPECT(O::relative_error(so, to_oracle(sd)) <= 1e-13, "formal_sum / scaled");

        // GaussianStream + draw_gaussian_factors + append_gaussian_columns (sketch.hpp:13-29)
        T::GaussianStream st(11);
        O::FactorRng ro(O::RngMode::Xoshiro, 11);
        T::GaussianFactorSet f = T::draw_gaussian_factors(x, 2, 7, st);
        O::FactorSet fo = O::draw_gaussian_factors(xo, 2, 7, ro);
        for (T::Index k = 2; k <= 6; ++k) EXPECT(bitwise(f.at_mode(k, 12), fo.at_mode(k)), "draw_gaussian_factors");
        T::append_gaussian_columns(f, 3, st);
        for (T::Index k = 2; k <= 6; ++k) {  // sketch.cpp:58-65: one stream.matrix(n_k, extra) per factor, in order
            O::Matrix extra = ro.draw(k, 12, 3, 0);
            O::Matrix& m = fo.factors[static_cast<std::size_t>(k - 2)];
            O::Matrix grown(m.rows, m.cols + 3);
            std::copy(m.a.begin(), m.a.end(), grown.a.begin());
            std::copy(extra.a.begin(), extra.a.end(), grown.a.begin() + static_cast<std::ptrdiff_t>(m.a.size()));
            m = grown;
        }
        for (T::Index k = 2; k <= 6; ++k) EXPECT(bitwise(f.at_mode(k, 12), fo.at_mode(k)), "append_gaussian_columns");

        // krp_partial_contractions_rl + append_krp_contractions (sketch.hpp:35-53)
        T::PartialContractionSet w = T::krp_partial_contractions_rl(x, f);
        O::ContractionSet wo = O::krp_partial_contractions_rl(xo, fo);
        for (T::Index k = 2; k <= 6; ++k) EXPECT(max_rel(w.at_mode(k), wo.at_mode(k)) <= 1e-12, "krp_partial_contractions_rl");
        T::GaussianFactorSet fresh = T::draw_gaussian_factors(x, 4, 4, st);
        O::FactorSet fresh_o = O::draw_gaussian_factors(xo, 4, 4, ro);
        T::append_krp_contractions(w, x, fresh);
        O::append_krp_contractions(wo, xo, fresh_o);
        for (T::Index k = 2; k <= 6; ++k) EXPECT(max_rel(w.at_mode(k), wo.at_mode(k)) <= 1e-12, "append_krp_contractions");
        EXPECT(w.at_mode(3).cols() == 10 && w.at_mode(4).cols() == 14, "append widths (lower modes keep theirs)");

        // generate_residual_sketch + residual_norm_estimate (round_rand.hpp:37-39, sketch.hpp:67)
        T::GaussianStream st2(5);
        O::FactorRng ro2(O::RngMode::Xoshiro, 5);
        T::PartialContractionSet w2 = T::krp_partial_contractions_rl(x, T::draw_gaussian_factors(x, 2, 5, st2));
        O::ContractionSet w2o = O::krp_partial_contractions_rl(xo, O::draw_gaussian_factors(xo, 2, 5, ro2));
        const O::Matrix zo = xo.core(1).vertical();  // (r_1 n) x r_2, the mode-2 unfolding
        T::Matrix z(zo.rows, zo.cols);
        z.a = zo.a;
        const O::Matrix qo = O::linalg::thin_qr_q(O::linalg::mul(zo, w2o.at_mode(3).left_cols(2)));
        T::Matrix q(qo.rows, qo.cols);
        q.a = qo.a;
        // mode k = 2: W_3 has 5 columns, used 2 + b 4 > 5 -> fresh factors for modes 3..d are drawn
        T::Matrix s = T::generate_residual_sketch(x, z, q, w2, 2, 4, st2);
        O::Matrix sref = O::generate_residual_sketch(xo, zo, qo, w2o, 2, 4, ro2);
        EXPECT(max_rel(s, sref) <= 1e-12, "generate_residual_sketch");
        for (T::Index k = 2; k <= 6; ++k) EXPECT(max_rel(w2.at_mode(k), w2o.at_mode(k)) <= 1e-12, "residual sketch appends");
        const double est = T::residual_norm_estimate(s, 4), est_o = O::residual_norm_estimate(sref, 4);
        EXPECT(std::abs(est - est_o) <= 1e-12 * (1 + est_o), "residual_norm_estimate");

        // rounding entry points with the reference's own stream (the layer's default)
        const O::TT fo_out = O::round_fixed_krp(xo, {6, 6, 6, 6, 6}, 7, O::RngMode::Xoshiro);
        const T::TTTensor fd = T::round_fixed_krp(x, {6, 6, 6, 6, 6}, 7);
        EXPECT(fd.ranks() == fo_out.ranks(), "round_fixed_krp ranks");
        EXPECT(O::relative_error(fo_out, to_oracle(fd)) <= 1e-10, "round_fixed_krp");
        O::AdaptiveConfig ac;
        ac.tolerance = 1e-4;
        ac.seed = 3;
        T::AdaptiveConfig tc;
        tc.tolerance = 1e-4;
        tc.seed = 3;
        const O::TT ao = O::round_adaptive_krp(xo, ac);
        const T::TTTensor ad = T::round_adaptive_krp(x, tc);
        EXPECT(ad.ranks() == ao.ranks(), "round_adaptive_krp ranks");
        EXPECT(O::relative_error(ao, to_oracle(ad)) <= 1e-10, "round_adaptive_krp");
        const O::TT dt = O::round_deterministic(xo, std::vector<O::Index>{4, 4, 4, 4, 4});
        const T::TTTensor dd = T::round_deterministic(x, std::vector<T::Index>{4, 4, 4, 4, 4});
        EXPECT(O::relative_error(dt, to_oracle(dd)) <= 1e-10, "round_deterministic");
        const double ne = T::estimate_norm_krp(x, 16, 21), ne_o = O::estimate_norm_krp(xo, 16, 21, O::RngMode::Xoshiro);
        EXPECT(std::abs(ne - ne_o) <= 1e-12 * ne_o, "estimate_norm_krp");

        // the TT-GMRES cookie harness (solver.hpp): the operator's factors, apply_operator,
        // and tt_gmres on the small cookie problem (test_solver.cpp:109-125)
        {
            const auto cp = T::build_cookie_problem(2, 8, 4, 1.0, 10.0);
            const auto co = O::build_cookie_problem(2, 8, 4, 1.0, 10.0);
            bool same = cp.op.num_terms() == co.op.num_terms();
            for (T::Index i = 0; same && i < cp.op.num_terms(); ++i)
                for (T::Index k = 0; k < cp.op.order(); ++k)
                    same = same && bitwise(cp.op.terms[static_cast<std::size_t>(i)][static_cast<std::size_t>(k)],
                                           co.op.terms[static_cast<std::size_t>(i)][static_cast<std::size_t>(k)]);
            EXPECT(same, "build_cookie_problem factors");
            EXPECT(O::relative_error(co.rhs, to_oracle(cp.rhs)) <= 1e-14, "build_cookie_problem rhs");
            const O::TT xr = O::random_gaussian_tt({64, 4, 4}, {1, 3, 2, 1}, 31);
            const auto ad2 = T::apply_operator(cp.op, to_device(xr));
            const auto ao2 = O::apply_operator(co.op, xr);
            bool ok = ad2.terms.size() == ao2.size();
            for (std::size_t i = 0; ok && i < ao2.size(); ++i) ok = O::relative_error(ao2[i], to_oracle(ad2.terms[i])) <= 1e-13;
            EXPECT(ok, "apply_operator");
            T::GMRESConfig gc;
            gc.rel_tolerance = 1e-5;
            gc.max_iterations = 120;
            gc.strategy = T::RoundingStrategy::AdaptiveKRPSum;
            gc.seed = 4;
            O::GmresConfig go;
            go.rel_tolerance = 1e-5;
            go.max_iterations = 120;
            go.strategy = O::GmresStrategy::AdaptiveKRPSum;
            go.seed = 4;
            const auto gd = T::tt_gmres(cp.op, cp.rhs, gc);
            const auto gr = O::tt_gmres(co.op, co.rhs, go);
            EXPECT(gd.converged && gr.converged && gd.iterations == gr.iterations, "tt_gmres iterations");
            EXPECT(gd.max_rank_history.size() == gr.max_rank_history.size() &&
                       std::equal(gd.max_rank_history.begin(), gd.max_rank_history.end(), gr.max_rank_history.begin()),
                   "tt_gmres rank history");
            EXPECT(O::relative_error(gr.solution, to_oracle(gd.solution)) <= 1e-8, "tt_gmres solution");
        }

        // the TTTensor constructor's checks, in the reference's order (tensor.cpp:66-79)
        EXPECT(errc_of([] { T::TTTensor(std::vector<T::Core>{}); }) == T::Errc::EmptyCoreList, "EmptyCoreList");
        EXPECT(errc_of([] { T::TTTensor({T::Core(2, 3, 1)}); }) == T::Errc::BoundaryRankNotOne, "BoundaryRankNotOne");
        EXPECT(errc_of([] { T::TTTensor({T::Core(1, 3, 2), T::Core(3, 3, 1)}); }) == T::Errc::RankChainMismatch,
               "RankChainMismatch");
        EXPECT(errc_of([] {
                   T::Core c(1, 3, 1);
                   c(0, 1, 0) = std::nan("");
                   T::TTTensor({c});
               }) == T::Errc::InvalidArgument,
               "non-finite core");
        EXPECT(errc_of([] { T::Core(0, 3, 1); }) == T::Errc::InvalidArgument, "core dimensions");
        EXPECT(errc_of([&] { T::draw_gaussian_factors(x, 1, 3, st); }) == T::Errc::InvalidArgument, "start mode");
        EXPECT(errc_of([&] { T::residual_norm_estimate(s, 0); }) == T::Errc::InvalidArgument, "block >= 1");

        if (g_fail) return 10;
        std::printf("dropin ok: every mirrored entry point matches the oracle\n");
        return 0;
    } catch (const T::Error& e) {
        std::printf("error: %s (errc %d status %d)\n", e.what(), static_cast<int>(e.code()), e.status());
        return 1;
    } catch (const O::Error& e) {
        std::printf("oracle error: %s\n", e.what());
        return 2;
    }
}
