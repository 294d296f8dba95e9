// tables.cpp — per-(N, mode) CRT constant tables, built natively at first use
// and cached immutably, mirroring the reference's registry
//   build_table  /root/reference/proj/include/oz2/moduli.hpp:93-142
//   table_for    moduli.hpp:145-153 (mutex-guarded, built once)
//   p_prime_fp32 mp.hpp:67-85, scaling_coeff_fp32 mp.hpp:89-93
// without GMP/MPFR: P <= prod(49 moduli) < 2^392 fits a fixed 512-bit integer,
// every conversion to fp64 is done with explicit round-to-nearest-even on the
// exact integer, and P' is bracketed in 64-bit extended precision (the
// reference brackets in MPFR; both reject an ambiguous rounding).
//
// Also builds the scaling-exponent step table used on the device: the
// reference's shift(c) = floor(fma_fp32(coeff, log2f(max(1, RU32(c))), P', Down))
// (scaling.hpp:159-194) is a monotone step function of the integer clearance
// maximum c, so the device evaluates it by counting thresholds — bit-identical
// to the reference by construction, with this host's libm log2 (the same libm
// the reference calls, softfp.hpp:147-150).
#include "tables.h"

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

namespace oz2g {

namespace {

// Fixed-width unsigned integer, little-endian 64-bit limbs.
struct Big {
    static constexpr int L = 8;
    uint64_t w[L] = {0, 0, 0, 0, 0, 0, 0, 0};

    static Big of(uint64_t v) { Big b; b.w[0] = v; return b; }
    bool is_zero() const { for (int i = 0; i < L; ++i) if (w[i]) return false; return true; }
    int bitlen() const {
        for (int i = L - 1; i >= 0; --i)
            if (w[i]) return 64 * i + (64 - __builtin_clzll(w[i]));
        return 0;
    }
    bool bit(int i) const { return (w[i >> 6] >> (i & 63)) & 1u; }
    void mul_small(uint64_t x) {
        unsigned __int128 carry = 0;
        for (int i = 0; i < L; ++i) {
            unsigned __int128 t = (unsigned __int128)w[i] * x + carry;
            w[i] = (uint64_t)t;
            carry = t >> 64;
        }
        if (carry) throw std::logic_error("oz2g tables: bignum overflow");
    }
    uint64_t divmod_small(uint64_t d) {  // *this /= d, returns remainder
        unsigned __int128 rem = 0;
        for (int i = L - 1; i >= 0; --i) {
            unsigned __int128 cur = (rem << 64) | w[i];
            w[i] = (uint64_t)(cur / d);
            rem = cur % d;
        }
        return (uint64_t)rem;
    }
    uint64_t mod_small(uint64_t d) const { Big t = *this; return t.divmod_small(d); }
    Big shr(int s) const {
        Big r;
        const int ls = s >> 6, bs = s & 63;
        for (int i = 0; i < L; ++i) {
            const int j = i + ls;
            if (j >= L) break;
            uint64_t v = w[j] >> bs;
            if (bs && j + 1 < L) v |= w[j + 1] << (64 - bs);
            r.w[i] = v;
        }
        return r;
    }
    Big shl(int s) const {
        Big r;
        const int ls = s >> 6, bs = s & 63;
        for (int i = L - 1; i >= 0; --i) {
            const int j = i - ls;
            if (j < 0) continue;
            uint64_t v = w[j] << bs;
            if (bs && j - 1 >= 0) v |= w[j - 1] >> (64 - bs);
            r.w[i] = v;
        }
        return r;
    }
    int cmp(const Big& o) const {
        for (int i = L - 1; i >= 0; --i)
            if (w[i] != o.w[i]) return w[i] < o.w[i] ? -1 : 1;
        return 0;
    }
    Big sub(const Big& o) const {  // requires *this >= o
        Big r;
        uint64_t borrow = 0;
        for (int i = 0; i < L; ++i) {
            const uint64_t a = w[i], b = o.w[i];
            const uint64_t d = a - b - borrow;
            borrow = (a < b) || (a - b < borrow) ? 1 : 0;
            r.w[i] = d;
        }
        return r;
    }
    // Round-to-nearest-even conversion to fp64 (exact for <= 53 bits).
    double to_double() const {
        const int bl = bitlen();
        if (bl == 0) return 0.0;
        if (bl <= 53) {
            uint64_t v = w[0];
            return (double)v;  // exact
        }
        const int drop = bl - 53;
        Big top = shr(drop);
        uint64_t mant = top.w[0];
        const bool half = bit(drop - 1);
        bool sticky = false;
        for (int i = 0; i < drop - 1 && !sticky; ++i) sticky = bit(i);
        if (half && (sticky || (mant & 1))) ++mant;  // may carry to 2^53: still exact
        return std::ldexp((double)mant, drop);
    }
    static Big from_double_int(double d) {  // d >= 0, integral
        int e;
        const double f = std::frexp(d, &e);
        const uint64_t mant = (uint64_t)std::ldexp(f, 53);
        Big b = Big::of(mant);
        const int sh = e - 53;
        return sh >= 0 ? b.shl(sh) : b.shr(-sh);
    }
    std::string to_dec() const {
        if (is_zero()) return "0";
        Big t = *this;
        std::string out;
        while (!t.is_zero()) {
            uint64_t r = t.divmod_small(10000000000000000000ull);
            char buf[32];
            if (t.is_zero()) snprintf(buf, sizeof buf, "%llu", (unsigned long long)r);
            else snprintf(buf, sizeof buf, "%019llu", (unsigned long long)r);
            out = std::string(buf) + out;
        }
        return out;
    }
};

constexpr int kModuli[49] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211,
                             199, 197, 193, 191, 181, 179, 173, 167, 163, 157, 151, 149, 139,
                             137, 131, 127, 113, 109, 107, 103, 101, 97,  89,  83,  79,  73,
                             71,  67,  61,  59,  53,  47,  43,  41,  37,  29};

long mod_inverse(long a, long p) {  // moduli.hpp:41-55
    long r0 = p, r1 = a % p, t0 = 0, t1 = 1;
    while (r1 != 0) {
        const long q = r0 / r1;
        r0 -= q * r1; std::swap(r0, r1);
        t0 -= q * t1; std::swap(t0, t1);
    }
    if (r0 != 1) throw std::domain_error("mod_inverse: inputs not coprime");
    if (t0 < 0) t0 += p;
    return t0;
}

// moduli.hpp:60-69 split_upper_bits
std::pair<double, double> split_upper_bits(const Big& x, int beta) {
    const int len = x.bitlen();
    const int shift = len - beta;
    if (shift <= 0) return {x.to_double(), 0.0};
    const Big head = x.shr(shift).shl(shift);
    const Big rem = x.sub(head);
    return {head.to_double(), rem.to_double()};
}

// RN(1/P) by binary long division (moduli.hpp:117, mp.hpp:59-62).
double reciprocal_rn(const Big& P) {
    const int b = P.bitlen();               // 2^(b-1) <= P < 2^b, P not a power of two
    Big R = Big::of(1).shl(b - 1);          // X = 2^(b-1)/P in (1/2, 1)
    uint64_t Q = 0;
    for (int i = 0; i < 56; ++i) {          // 56 fractional bits of X
        R = R.shl(1);
        Q <<= 1;
        if (R.cmp(P) >= 0) { R = R.sub(P); Q |= 1; }
    }
    const bool sticky = !R.is_zero();
    uint64_t mant = Q >> 3;                 // 53 bits
    const uint64_t low = Q & 7;
    if (low > 4 || (low == 4 && (sticky || (mant & 1)))) ++mant;  // RN, ties to even
    return std::ldexp((double)mant, -(56 - 3) - (b - 1));
}

float round_down_f32(long double v) {
    float f = (float)v;
    if ((long double)f > v) f = std::nextafterf(f, -INFINITY);
    return f;
}

// mp.hpp:67-85: RD32(log2(P-1)/2 - 0.5), bracketed.
float p_prime_fp32(const Big& P) {
    const Big pm1 = P.sub(Big::of(1));
    const int bl = pm1.bitlen();
    long double l2;
    if (bl <= 64) {
        l2 = log2l((long double)pm1.w[0]);
    } else {
        const int s = bl - 64;
        const Big top = pm1.shr(s);
        const Big rest = pm1.sub(top.shl(s));
        // log2(top*2^s + rest) = s + log2(top) + log2(1 + rest/(top*2^s)); rest < 2^s
        const long double frac = (long double)rest.to_double() / std::ldexp((long double)top.w[0], s);
        l2 = (long double)s + log2l((long double)top.w[0]) + log1pl(frac) / logl(2.0L);
    }
    const long double v = l2 / 2.0L - 0.5L;
    const long double eps = 1e-15L;  // >> the extended-precision error of v (|v| < 200)
    const float lo = round_down_f32(v - eps), hi = round_down_f32(v + eps);
    if (lo != hi) throw std::runtime_error("p_prime_fp32: bracketing did not converge");
    return lo;
}

// mp.hpp:89-93: RD32(-2^21/(2^22-1)) = -0x1.000006p-1.
constexpr float kScalingCoeff = -0x1.000006p-1f;

}  // namespace

// softfp.hpp:153-159 fp32_round_up
float fp32_round_up(int64_t v) {
    float f = (float)v;
    if ((double)f < (double)v) f = std::nextafterf(f, INFINITY);
    return f;
}

// scaling.hpp:159-194 for one clearance maximum c: floor(RD32(coeff*e + P')).
// For |coeff*e + P'| < 2^24 every integer is a binary32 value, hence
// floor(RD32(v)) == floor(v) and the exact real floor is evaluated: coeff*e is
// exact in fp64 (24x24 bits) and TwoSum makes the sum exact as hi + lo.
int shift_of_cmax(float p_prime, int64_t c, float* e_out) {
    const float d = fp32_round_up(c);
    const float mx = d > 1.0f ? d : 1.0f;
    const float e = (float)std::log2((double)mx);  // log2_fp32, softfp.hpp:147-150
    if (e_out) *e_out = e;
    const double prod = (double)kScalingCoeff * (double)e;
    const double pp = (double)p_prime;
    const double hi = prod + pp;
    const double bb = hi - prod;
    const double lo = (prod - (hi - bb)) + (pp - bb);
    double fl = std::floor(hi);
    if (fl == hi && lo < 0.0) fl -= 1.0;
    return (int)fl;
}

static Table build_table(int n, int mode) {
    if (n < 2 || n > kMaxModuli) throw std::domain_error("build_table: N out of [2, 49]");
    Table t;
    t.n = n;
    t.mode = mode;
    Big P = Big::of(1);
    for (int l = 0; l < n; ++l) {
        t.p[l] = kModuli[l];
        P.mul_small((uint64_t)kModuli[l]);
        t.rho += kModuli[l] / 2;
    }
    Big r[kMaxModuli];
    int max_log2r = 0;
    for (int l = 0; l < n; ++l) {
        Big m = P;
        m.divmod_small((uint64_t)t.p[l]);
        t.q[l] = (int)mod_inverse((long)m.mod_small((uint64_t)t.p[l]), t.p[l]);
        r[l] = m;
        r[l].mul_small((uint64_t)t.q[l]);
        if (r[l].bitlen() - 1 > max_log2r) max_log2r = r[l].bitlen() - 1;
    }
    t.P1 = P.to_double();
    if (mode == kF64) {
        const Big p1 = Big::from_double_int(t.P1);
        t.P2 = P.cmp(p1) >= 0 ? P.sub(p1).to_double() : -p1.sub(P).to_double();
    }
    t.P_inv = reciprocal_rn(P);
    if (mode == kF64) {
        int clr = 0;
        while ((1l << clr) < t.rho) ++clr;
        for (int l = 0; l < n; ++l) {
            const int log2r = r[l].bitlen() - 1;
            const int b = 53 - clr + log2r - max_log2r;
            t.beta[l] = b;
            const auto hs = split_upper_bits(r[l], b);
            t.s1[l] = hs.first;
            t.s2[l] = hs.second;
        }
    } else {
        for (int l = 0; l < n; ++l) t.s1[l] = r[l].to_double();
    }
    t.P_prime = p_prime_fp32(P);
    t.P_dec = P.to_dec();

    // Step table of shift(c) over every reachable clearance maximum c in
    // [0, 2^29] (entries <= 2^12 k and k <= 2^17, int8gemm.hpp:12).
    const int64_t cmax = int64_t(1) << 29;
    t.shift0 = shift_of_cmax(t.P_prime, 0, nullptr);
    const int slast = shift_of_cmax(t.P_prime, cmax, nullptr);
    for (int target = t.shift0 - 1; target >= slast; --target) {
        int64_t lo = 0, hi = cmax;  // shift(lo) > target, shift(hi) <= target
        while (hi - lo > 1) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (shift_of_cmax(t.P_prime, mid, nullptr) <= target) hi = mid; else lo = mid;
        }
        if (t.nthr >= (int)(sizeof(t.thr) / sizeof(t.thr[0]))) throw std::logic_error("step table overflow");
        t.thr[t.nthr++] = (int32_t)hi;
    }
    return t;
}

const Table& table_for(int n, int mode) {
    static std::map<std::pair<int, int>, Table> cache;
    static std::mutex mtx;
    std::lock_guard<std::mutex> lock(mtx);
    const auto key = std::make_pair(n, mode);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, build_table(n, mode)).first;
    return it->second;
}

// Upward-rounded fp64 image of a positive extended-precision value whose
// relative error is far below 2^-60: round to nearest, then step up twice.
static double up2(long double v) {
    double d = (double)v;
    d = std::nextafter(d, INFINITY);
    return std::nextafter(d, INFINITY);
}

BoundScalars bound_scalars(const Table& t, int64_t k) {
    // P and rho as extended precision (relative error 2^-64)
    long double P = 0.0L;
    for (char ch : t.P_dec) P = P * 10.0L + (long double)(ch - '0');
    const long double rho = (long double)t.rho;
    const long double u64 = 0x1p-53L, u32 = 0x1p-24L;
    BoundScalars b;
    const long double denom = 32.0L * (P - 1.0L);
    b.t_up = up2(1.0L / sqrtl(denom));   // bounds.hpp:132-141
    b.t2_up = up2(1.0L / denom);
    long double rc;                      // bounds.hpp:74-81
    if (t.mode == kF32) {
        rc = (1.0L + u32) * (long double)(t.n + 2) * u64 * rho * P;
        b.ucoef = 0x1p-24;
    } else {
        int clr = 0;
        while ((1l << clr) < t.rho) ++clr;
        rc = (1.0L + 3.0L * u64) * ldexpl(1.0L, 1 + clr) * (long double)(t.n + 2) * u64 * u64 * rho * P;
        b.ucoef = 3.0 * 0x1p-53;
    }
    b.rconst_up = up2(rc);
    b.kpr_cheap_up = up2((long double)k + rc + (long double)b.ucoef * P / 2.0L);  // bounds.hpp:89-92, :201
    b.k_rconst_up = up2((long double)k + rc);
    return b;
}

int fp32_safe_moduli_max() {  // moduli.hpp:157-170
    static const int value = [] {
        const Big limit = Big::of((1u << 24) - 1).shl(105);
        Big prod = Big::of(1);
        int cnt = 0;
        for (int pl : kModuli) {
            prod.mul_small((uint64_t)pl);
            if (prod.cmp(limit) > 0) break;
            ++cnt;
        }
        return cnt;
    }();
    return value;
}

}  // namespace oz2g
