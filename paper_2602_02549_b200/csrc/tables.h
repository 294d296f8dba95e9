// tables.h — host-side constant registry (see tables.cpp).
#pragma once
#include <cstdint>
#include <string>

namespace oz2g {

constexpr int kMaxModuli = 49;
constexpr int kF32 = 0, kF64 = 1;

// ModuliTable (moduli.hpp:78-91) minus the mpz members, plus the device
// step table for the scaling exponents.
struct Table {
    int n = 0, mode = kF64;
    int p[kMaxModuli] = {}, q[kMaxModuli] = {}, beta[kMaxModuli] = {};
    double s1[kMaxModuli] = {}, s2[kMaxModuli] = {};
    long rho = 0;
    double P1 = 0, P2 = 0, P_inv = 0;
    float P_prime = 0;
    std::string P_dec;
    int shift0 = 0, nthr = 0;
    int32_t thr[64] = {};
};

const Table& table_for(int n, int mode);  // throws std::domain_error for N outside [2, 49]

// Scalars of the deterministic error bounds (bounds.hpp:71-92, :132-141),
// every one rounded upward (u_coef and 1 - u_coef are exact).
struct BoundScalars {
    double t_up;         // >= 1 / sqrt(2^5 (P - 1))
    double t2_up;        // >= 1 / (2^5 (P - 1))
    double rconst_up;    // >= r_const (R_b without the u|A'B'| term)
    double ucoef;        // u_coef: 2^-24 (fp32) or 3 * 2^-53 (fp64)
    double kpr_cheap_up; // >= k + r_const + u_coef * P / 2
    double k_rconst_up;  // >= k + r_const
};
BoundScalars bound_scalars(const Table& t, int64_t k);
int fp32_safe_moduli_max();
float fp32_round_up(int64_t v);
int shift_of_cmax(float p_prime, int64_t c, float* e_out);

}  // namespace oz2g
