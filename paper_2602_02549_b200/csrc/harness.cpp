// harness.cpp — host-side pieces of the reference's experiment harness that
// the library exposes for callers:
//   the synthetic-matrix stream   prng.hpp:1-54 / gen.hpp:15-31
//   derive_seed                   experiment.hpp:83-88
// The stream is a fixed specification (xoshiro256** seeded by four
// splitmix64 outputs; uniform = ((next >> 11) + 1) * 2^-53 on (0, 1];
// Box-Muller normal from two fresh uniforms; entries (u - 1/2) exp(g phi),
// redrawn while zero or non-finite in the working precision), so the same
// seed yields the reference's matrices bit for bit with the same libm.
#include <cmath>
#include <cstdint>

#include "../../include/oz2g.h"

namespace {

struct SplitMix {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
};

class Xoshiro {
public:
    explicit Xoshiro(uint64_t seed) {
        SplitMix sm{seed};
        for (uint64_t& w : st_) w = sm.next();
    }
    uint64_t next() {
        const uint64_t out = rotl(st_[1] * 5, 7) * 9;
        const uint64_t t = st_[1] << 17;
        st_[2] ^= st_[0];
        st_[3] ^= st_[1];
        st_[1] ^= st_[2];
        st_[0] ^= st_[3];
        st_[2] ^= t;
        st_[3] = rotl(st_[3], 45);
        return out;
    }
    double uniform() { return (double)((next() >> 11) + 1) * 0x1p-53; }  // (0, 1]
    double normal() {
        const double u1 = uniform(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
    }

private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t st_[4];
};

template <class T>
void fill(int64_t rows, int64_t cols, double phi, uint64_t seed, T* out) {
    Xoshiro rng(seed);
    for (int64_t e = 0; e < rows * cols; ++e) {
        T v;
        do {
            const double u = rng.uniform();
            const double g = rng.normal();
            v = (T)((u - 0.5) * std::exp(g * phi));
        } while (v == T(0) || !std::isfinite((double)v));
        out[e] = v;
    }
}

}  // namespace

extern "C" {

int oz2g_gen_matrix(int prec, int64_t rows, int64_t cols, double phi, uint64_t seed, void* out) {
    if (!(phi >= 0)) return OZ2G_DOMAIN_ERROR;  // gen.hpp:17
    if (rows < 0 || cols < 0) return OZ2G_INVALID_ARGUMENT;
    if (prec == OZ2G_FP64) fill(rows, cols, phi, seed, (double*)out);
    else if (prec == OZ2G_FP32) fill(rows, cols, phi, seed, (float*)out);
    else return OZ2G_INVALID_ARGUMENT;
    return OZ2G_OK;
}

uint64_t oz2g_derive_seed(uint64_t seed, uint64_t trial, uint64_t role) {  // experiment.hpp:83-88
    SplitMix s{seed};
    (void)s.next();
    s.s ^= 0x5851f42d4c957f2dull * (trial + 1) + 0x14057b7ef767814full * (role + 1);
    return s.next();
}

}  // extern "C"
