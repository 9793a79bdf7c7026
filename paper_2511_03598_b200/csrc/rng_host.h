// rng_host.h — the reference's sequential Gaussian stream, for the library's
// XOSHIRO compatibility mode (factors drawn on the host in the reference's
// order and uploaded). Restates proj/core/src/rng.cpp:11-78: splitmix64
// seeding, xoshiro256++ uniforms, Box-Muller pairs with a cached spare.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

namespace ttr {

inline std::uint64_t splitmix64(std::uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {
    std::uint64_t s = seed ^ (0xd1342543de82ef95ULL * (tag + 1));
    return splitmix64(s);
}

class XoshiroGauss {
public:
    explicit XoshiroGauss(std::uint64_t seed) {
        std::uint64_t s = seed;
        for (auto& w : s_) w = splitmix64(s);
    }
    double next() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * M_PI * u2;
        spare_ = radius * std::sin(angle);
        has_spare_ = true;
        return radius * std::cos(angle);
    }
    // rows x cols, column-major (rng.cpp:62-67)
    std::vector<double> matrix(std::int64_t rows, std::int64_t cols) {
        std::vector<double> m(static_cast<std::size_t>(rows * cols));
        for (auto& v : m) v = next();
        return m;
    }

private:
    static std::uint64_t rotl(std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    double uniform() {
        const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
        const std::uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return static_cast<double>(result >> 11) * 0x1.0p-53;
    }
    std::uint64_t s_[4];
    double spare_ = 0.0;
    bool has_spare_ = false;
};

}  // namespace ttr
