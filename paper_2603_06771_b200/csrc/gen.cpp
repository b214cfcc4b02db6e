// gen.cpp -- seeded synthetic clouds (host).  Inputs only, not on the measured path.
//
// Draw order and formulas follow the reference's generator helpers (rng.hpp:18-58,
// io.cpp:122-130) so the uniform clouds (cfg0, cfg4) are the reference's own; the terrain and
// mixed clouds (cfg1-3) are the SURVEY.md §8d definitions built on the same helpers.  Built
// without FMA contraction (-ffp-contract=off) so both the CPU baseline and the GPU path see
// identical arrays.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/linoct_b200.h"

namespace {

double unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

std::uint64_t below(std::mt19937_64& g, std::uint64_t n) {
    if (n <= 1) return 0;
    const int bits = 64 - std::countl_zero(n - 1);
    const std::uint64_t mask = bits == 64 ? ~0ull : ((1ull << bits) - 1);
    for (;;) {
        const std::uint64_t x = g() & mask;
        if (x < n) return x;
    }
}

double normal(std::mt19937_64& g) {
    double u1 = unit(g);
    while (u1 <= 0.0) u1 = unit(g);
    const double u2 = unit(g);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
}

void terrain(std::mt19937_64& g, std::uint64_t n, double extent, double* xyz) {
    for (std::uint64_t i = 0; i < n; ++i) {
        const double x = unit(g) * extent;
        const double y = unit(g) * extent;
        const double s = 10.0 * std::sin(x / 50.0) * std::cos(y / 70.0);
        xyz[3 * i] = x;
        xyz[3 * i + 1] = y;
        xyz[3 * i + 2] = s + 0.1 * normal(g);
    }
}

}  // namespace

extern "C" {

int lo_generate_uniform(uint64_t n, uint64_t seed, double extent, double* xyz) {
    std::mt19937_64 g(seed);
    for (uint64_t i = 0; i < 3 * n; ++i) xyz[i] = unit(g) * extent;
    return LO_OK;
}

int lo_generate_terrain(uint64_t n, uint64_t seed, double extent_xy, double* xyz) {
    std::mt19937_64 g(seed);
    terrain(g, n, extent_xy, xyz);
    return LO_OK;
}

int lo_generate_mixed(uint64_t n, uint64_t seed, double* xyz) {
    std::mt19937_64 g(seed);
    const uint64_t nt = n * 7 / 10, nc = n * 2 / 10, nn = n - nt - nc;
    terrain(g, nt, 3000.0, xyz);
    double lo[3] = {0, 0, 0}, hi[3] = {3000, 3000, 3000};
    if (nt) {
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = xyz[a];
        for (uint64_t i = 0; i < nt; ++i)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], xyz[3 * i + a]);
                hi[a] = std::max(hi[a], xyz[3 * i + a]);
            }
    }
    std::vector<double> centres(3000);
    for (int c = 0; c < 1000; ++c)
        for (int a = 0; a < 3; ++a) centres[3 * c + a] = lo[a] + unit(g) * (hi[a] - lo[a]);
    double* p = xyz + 3 * nt;
    for (uint64_t i = 0; i < nc; ++i) {
        const double* c = &centres[3 * below(g, 1000)];
        p[3 * i] = c[0] + 2.0 * normal(g);
        p[3 * i + 1] = c[1] + 2.0 * normal(g);
        p[3 * i + 2] = c[2] + 2.0 * normal(g);
    }
    p += 3 * nc;
    for (uint64_t i = 0; i < nn; ++i) {
        p[3 * i] = unit(g) * 3000.0;
        p[3 * i + 1] = unit(g) * 3000.0;
        p[3 * i + 2] = -20.0 + unit(g) * 80.0;
    }
    return LO_OK;
}

int lo_sample_indices(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out) {
    std::vector<uint32_t> pool(n);
    for (uint32_t i = 0; i < n; ++i) pool[i] = i;
    std::mt19937_64 g(seed);
    const uint32_t take = std::min(k, n);
    for (uint32_t i = 0; i < take; ++i) std::swap(pool[i], pool[i + below(g, n - i)]);
    std::copy(pool.begin(), pool.begin() + take, out);
    return LO_OK;
}

}  // extern "C"
