// C++ drop-in check: the reference's own emulate tests (test_emulate.cpp),
// written against oz2::os_ii<T> from include/oz2g/emulate.hpp — the same
// source a reference user compiles, now running on the B200 library.
#include <oz2g/emulate.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>

static int failures = 0;
#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++failures; } \
    } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

int main() {
    using namespace oz2;
    // test_emulate.cpp:13-20 — 1x1 unit product, exact at N=2
    Matrix<double> one(1, 1, 1.0);
    CHECK(os_ii(one, one, 2).C(0, 0) == 1.0);
    Matrix<float> onef(1, 1, 1.0f);
    CHECK(os_ii(onef, onef, 2).C(0, 0) == 1.0f);
    const auto tr = os_ii(one, one, 2, true);
    CHECK(tr.scaling.mu[0] == 7 && tr.scaling.nu[0] == 7);
    CHECK(tr.crt.W.size() == 2 && tr.crt.W[0](0, 0) == 0 && tr.crt.W[1](0, 0) == 64);
    CHECK(tr.crt.C1(0, 0) == 16384.0 && tr.crt.Q(0, 0) == 0.0);
    // :25-30
    for (int n : {10, 30, 49}) CHECK(std::abs(os_ii(one, one, n).C(0, 0) - 1.0) <= 0x1p-40);
    for (int n : {10, 16}) CHECK(std::abs(static_cast<double>(os_ii(onef, onef, n).C(0, 0)) - 1.0) <= 0x1p-18);
    // :67-73 fp32 range error beyond the ceiling
    Matrix<float> a3(3, 8), b3(8, 3);
    for (int i = 0; i < 24; ++i) { a3.data()[i] = 0.25f + 0.01f * i; b3.data()[i] = -0.5f + 0.03f * i; }
    CHECK(throws_as<std::range_error>([&] { os_ii(a3, b3, fp32_safe_moduli_max() + 1, false); }));
    // :102-111 intermediates dropped unless requested
    const auto lean = os_ii(one, one, 5, false);
    CHECK(lean.crt.W.empty() && lean.crt.C1.empty() && lean.scaling.Aprime.empty());
    const auto full = os_ii(one, one, 5, true);
    CHECK(full.crt.W.size() == 5 && !full.scaling.Aprime.empty());
    // :113-120 preconditions
    Matrix<double> a(2, 3), b(3, 2);
    a(0, 0) = 1.0; a(0, 1) = 1.0; a(0, 2) = 1.0;
    for (int h = 0; h < 3; ++h) { b(h, 0) = 1.0; b(h, 1) = 1.0; }
    CHECK(throws_as<std::domain_error>([&] { os_ii(a, b, 5); }));
    Matrix<double> bad(4, 2, 1.0);
    CHECK(throws_as<std::invalid_argument>([&] { os_ii(a, bad, 5); }));
    // :89-100 power-of-two inverse scaling exact in the normal range
    Matrix<double> A(4, 12), B(12, 4);
    for (int i = 0; i < 48; ++i) { A.data()[i] = std::sin(1.0 + i) * 0.7; B.data()[i] = std::cos(2.0 + 3 * i) * 1.3; }
    const auto res = os_ii(A, B, 12, true);
    CHECK(!res.subnormal);
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            CHECK(std::ldexp(std::ldexp(res.C(i, j), res.scaling.mu[i]), res.scaling.nu[j]) == res.crt.Cpp64(i, j));
    // bounds.hpp:217-243 suggest_n (cheap, absolute) and the tight / relative search
    const auto sc = suggest_n(A, B, 1e-6);
    CHECK(sc.achievable && sc.n >= 2 && sc.bound_max <= 1e-6);
    CHECK(!suggest_n(A, B, 1e-300).achievable);
    const auto st = suggest_n_tight(A, B, 1e-13, true);
    CHECK(st.achievable && st.n >= 2 && st.bound_max <= 1e-13);
    CHECK(suggest_n_tight(A, B, 1e-13, false).n <= suggest_n(A, B, 1e-13).n || !suggest_n(A, B, 1e-13).achievable);
    CHECK(throws_as<std::domain_error>([&] { suggest_n(A, B, -1.0); }));
    // tuning options: a variant gives the same C; bad names / values throw
    {
        const auto base = os_ii(A, B, 12);
        set_option("gemm", 1);  // CTA-pair residue GEMM
        CHECK(get_option("gemm") == 1);
        const auto pair = os_ii(A, B, 12);
        set_option("gemm", 0);
        CHECK(std::memcmp(base.C.data(), pair.C.data(), sizeof(double) * 4 * 4) == 0);
        CHECK(throws_as<std::invalid_argument>([&] { set_option("gemm", 7); }));
        CHECK(throws_as<std::invalid_argument>([&] { get_option("no_such_option"); }));
    }
    // multi-device tiling (the device listed twice): C identical to os_ii
    {
        Matrix<double> X(40, 33), Y(33, 27);
        for (int i = 0; i < 40 * 33; ++i) X.data()[i] = std::sin(0.3 * i) * std::exp(0.01 * (i % 17));
        for (int i = 0; i < 33 * 27; ++i) Y.data()[i] = std::cos(0.7 * i) - 0.25;
        const auto single = os_ii(X, Y, 14);
        const auto tiled = os_ii_multi(X, Y, 14, {0, 0});
        CHECK(std::memcmp(single.C.data(), tiled.C.data(), sizeof(double) * 40 * 27) == 0);
        CHECK(throws_as<std::invalid_argument>([&] { os_ii_multi(X, Y, 14, {}); }));
    }
    // large call through the drop-in (pipelined host path even though the
    // scaling vectors are returned): same C as the device-pointer path
    {
        const std::int64_t m = 2304, k = 96, n = 300;
        Matrix<double> X(m, k), Y(k, n);
        for (std::int64_t i = 0; i < m * k; ++i) X.data()[i] = std::sin(0.001 * i) + 0.5 * std::cos(0.37 * i);
        for (std::int64_t i = 0; i < k * n; ++i) Y.data()[i] = std::cos(0.002 * i) - 0.1;
        const auto r = os_ii(X, Y, 16);
        CHECK(static_cast<std::int64_t>(r.scaling.mu.size()) == m && static_cast<std::int64_t>(r.scaling.nu.size()) == n);
        const auto t = os_ii_multi(X, Y, 16, {0});
        CHECK(std::memcmp(r.C.data(), t.C.data(), sizeof(double) * m * n) == 0);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
