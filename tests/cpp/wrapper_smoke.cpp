// Drop-in check of include/ttround_b200/ttround.hpp: the reference's calling
// code shape (tools/ttround_main.cpp:86-119 dispatch_rounding) compiled
// against the B200 library. Prints one line; exit code != 0 on failure.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ttround_b200/ttround.hpp"

using namespace ttround;

int main() {
    try {
        // d=2 rank-1 tensor of the reference's tiny KAT (tests/test_tensor.cpp:148-153)
        TTTensor tiny({2, 2}, {1, 1, 1}, {1.0, 2.0, 3.0, 4.0});
        const double nrm = norm_exact(tiny);
        if (std::abs(nrm - std::sqrt(125.0)) > 1e-12) return 2;
        // d=4 random-ish tensor, exact at full width
        std::vector<Index> n{5, 4, 5, 4}, r{1, 4, 5, 3, 1};
        std::vector<double> cores;
        for (std::size_t k = 0; k < n.size(); ++k)
            for (Index e = 0; e < r[k] * n[k] * r[k + 1]; ++e) cores.push_back(std::sin(0.37 * cores.size() + 1.0));
        TTTensor x(n, r, cores);
        TTTensor y = round_fixed_krp(x, {4, 5, 3}, 7);
        const double err = relative_error(x, y);
        AdaptiveConfig cfg;
        cfg.tolerance = 1e-8;
        cfg.seed = 3;
        TTTensor ya = round_adaptive_krp(x, cfg);
        TTTensor yd = round_deterministic(x, 1e-12);
        std::printf("wrapper ok: fixed err %.2e adaptive err %.2e det err %.2e\n", err, relative_error(x, ya),
                    relative_error(x, yd));
        try {
            round_fixed_krp(x, {0, 1, 1}, 0);
            return 3;
        } catch (const Error& e) {
            if (e.code() != Errc::InvalidRanks) return 4;
        }
        return err <= 1e-10 ? 0 : 5;
    } catch (const Error& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
}
