// oz2g/emulate.hpp — drop-in C++ interface for the reference's hot path,
// backed by the B200 library through the C ABI in oz2g.h.
//
// Mirrors, name for name:
//   oz2::Matrix<T>                 /root/reference/proj/include/oz2/matrix.hpp:11-49
//   oz2::ScalingOutput             scaling.hpp:20-28
//   oz2::CrtIntermediates          crt.hpp:81-87
//   oz2::EmulationResult<T>        emulate.hpp:17-24
//   oz2::os_ii<T>(a, b, n, keep)   emulate.hpp:54-88
//   oz2::fp32_safe_moduli_max()    moduli.hpp:157-170
// with the same exception classes (std::invalid_argument / domain_error /
// range_error / logic_error).  A reference user switches by including this
// header instead of <oz2/emulate.hpp> and linking liboz2g.so.  Differences:
// EmulationResult::table is an oz2g_table (no mpz members), and the library
// additionally returns the clearance maxima it computes on the device.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../oz2g.h"

namespace oz2 {

template <class T>
class Matrix {
public:
    Matrix() : rows_(0), cols_(0) {}
    Matrix(std::int64_t rows, std::int64_t cols, T init = T{})
        : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), init) {
        if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
    }
    std::int64_t rows() const { return rows_; }
    std::int64_t cols() const { return cols_; }
    std::int64_t size() const { return rows_ * cols_; }
    bool empty() const { return data_.empty(); }
    T& operator()(std::int64_t i, std::int64_t j) { return data_[static_cast<std::size_t>(i * cols_ + j)]; }
    const T& operator()(std::int64_t i, std::int64_t j) const { return data_[static_cast<std::size_t>(i * cols_ + j)]; }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
    friend bool operator==(const Matrix& a, const Matrix& b) {
        return a.rows_ == b.rows_ && a.cols_ == b.cols_ && a.data_ == b.data_;
    }

private:
    std::int64_t rows_, cols_;
    std::vector<T> data_;
};

using MatrixF32 = Matrix<float>;
using MatrixF64 = Matrix<double>;
using MatrixI8 = Matrix<std::int8_t>;
using MatrixI32 = Matrix<std::int32_t>;

inline void require_dims(bool ok, const std::string& what) {
    if (!ok) throw std::invalid_argument("dimension mismatch: " + what);
}

enum class Prec { F32, F64 };
template <class T>
inline constexpr Prec prec_of = std::is_same_v<T, float> ? Prec::F32 : Prec::F64;

struct ScalingOutput {
    Matrix<double> Aprime, Bprime;
    std::vector<std::int16_t> mu, nu, mu_prime, nu_prime;
    MatrixI32 Cbar;
    MatrixF32 Dbar;
    std::vector<float> e, f;
};

struct CrtIntermediates {
    std::vector<MatrixI8> W;
    Matrix<double> C1, C2, Q, Cpp64;
    MatrixF32 Cpp32;
};

template <class T>
struct EmulationResult {
    Matrix<T> C;
    ScalingOutput scaling;
    CrtIntermediates crt;
    oz2g_table table{};
    bool subnormal = false;
};

namespace detail {

inline void throw_status(int rc) {
    const std::string msg = oz2g_last_error();
    switch (rc) {
        case OZ2G_OK: return;
        case OZ2G_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case OZ2G_DOMAIN_ERROR: throw std::domain_error(msg);
        case OZ2G_RANGE_ERROR: throw std::range_error(msg);
        case OZ2G_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error("oz2g: " + msg);
    }
}

}  // namespace detail

inline int fp32_safe_moduli_max() { return oz2g_fp32_safe_moduli_max(); }

// emulate.hpp:54-88.  Runs on the current CUDA device with host matrices.
template <class T>
EmulationResult<T> os_ii(const Matrix<T>& a, const Matrix<T>& b, int n, bool keep_intermediates = false) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
    require_dims(a.cols() == b.rows(), "os_ii inner dimension");
    const std::int64_t m = a.rows(), k = a.cols(), nn = b.cols();
    const int prec = std::is_same_v<T, double> ? OZ2G_FP64 : OZ2G_FP32;
    EmulationResult<T> r;
    r.C = Matrix<T>(m, nn);
    oz2g_intermediates inter;
    std::memset(&inter, 0, sizeof inter);
    if (keep_intermediates && n >= 2 && n <= OZ2G_MAX_MODULI) {
        auto& s = r.scaling;
        s.mu.resize(m); s.nu.resize(nn); s.mu_prime.resize(m); s.nu_prime.resize(nn);
        s.e.resize(m); s.f.resize(nn);
        s.Aprime = Matrix<double>(m, k); s.Bprime = Matrix<double>(k, nn);
        s.Cbar = MatrixI32(m, nn); s.Dbar = MatrixF32(m, nn);
        inter.mu = s.mu.data(); inter.nu = s.nu.data(); inter.mu_prime = s.mu_prime.data();
        inter.nu_prime = s.nu_prime.data(); inter.e = s.e.data(); inter.f = s.f.data();
        inter.Aprime = s.Aprime.data(); inter.Bprime = s.Bprime.data();
        inter.Cbar = s.Cbar.data(); inter.Dbar = s.Dbar.data();
        auto& c = r.crt;
        std::vector<std::int8_t> w(static_cast<std::size_t>(n) * static_cast<std::size_t>(m * nn));
        c.C1 = Matrix<double>(m, nn); c.C2 = Matrix<double>(m, nn); c.Q = Matrix<double>(m, nn);
        c.Cpp64 = Matrix<double>(m, nn);
        inter.W = w.data(); inter.C1 = c.C1.data(); inter.C2 = c.C2.data(); inter.Q = c.Q.data();
        inter.Cpp64 = c.Cpp64.data();
        if (prec == OZ2G_FP32) { c.Cpp32 = MatrixF32(m, nn); inter.Cpp32 = c.Cpp32.data(); }
        oz2g_diag diag;
        detail::throw_status(oz2g_gemm(prec, m, nn, k, a.data(), k, b.data(), nn, r.C.data(), nn, n,
                                       OZ2G_HOST_PTRS, nullptr, &inter, &diag, nullptr, nullptr));
        r.subnormal = diag.subnormal != 0;
        c.W.assign(static_cast<std::size_t>(n), MatrixI8(m, nn));
        for (int l = 0; l < n; ++l)
            std::memcpy(c.W[l].data(), w.data() + static_cast<std::size_t>(l) * static_cast<std::size_t>(m * nn),
                        static_cast<std::size_t>(m * nn));
    } else {
        // keep == false keeps mu, nu, mu', nu', e, f like the reference (emulate.hpp:75-86)
        auto& s = r.scaling;
        if (n >= 2 && n <= OZ2G_MAX_MODULI) {
            s.mu.resize(m); s.nu.resize(nn); s.mu_prime.resize(m); s.nu_prime.resize(nn);
            s.e.resize(m); s.f.resize(nn);
            inter.mu = s.mu.data(); inter.nu = s.nu.data(); inter.mu_prime = s.mu_prime.data();
            inter.nu_prime = s.nu_prime.data(); inter.e = s.e.data(); inter.f = s.f.data();
        }
        oz2g_diag diag;
        detail::throw_status(oz2g_gemm(prec, m, nn, k, a.data(), k, b.data(), nn, r.C.data(), nn, n,
                                       OZ2G_HOST_PTRS, nullptr, &inter, &diag, nullptr, nullptr));
        r.subnormal = diag.subnormal != 0;
    }
    detail::throw_status(oz2g_table_for(n, prec, &r.table));
    return r;
}

// bounds.hpp:208-243: the smallest N whose cheap error bound (absolute) meets
// `target`, one clearance pass on the device.
struct SuggestResult {
    bool achievable = false;
    int n = 0;
    double bound_max = 0;
};

template <class T>
SuggestResult suggest_n(const Matrix<T>& a, const Matrix<T>& b, double target) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
    require_dims(a.cols() == b.rows(), "suggest_n inner dimension");
    const int prec = std::is_same_v<T, double> ? OZ2G_FP64 : OZ2G_FP32;
    SuggestResult r;
    detail::throw_status(oz2g_suggest_n(prec, a.rows(), b.cols(), a.cols(), a.data(), a.cols(), b.data(), b.cols(),
                                        target, OZ2G_HOST_PTRS, nullptr, &r.n, &r.bound_max));
    r.achievable = r.n > 0;
    return r;
}

// The same search with the TIGHT bound (bounds.hpp:182-195), absolute or
// relative to (|A||B|)_ij (oz2g_suggest_n_tight): the N the north star asks
// for ("N from the paper's bound for 1e-15 relative accuracy").
template <class T>
SuggestResult suggest_n_tight(const Matrix<T>& a, const Matrix<T>& b, double target, bool relative = true) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
    require_dims(a.cols() == b.rows(), "suggest_n inner dimension");
    const int prec = std::is_same_v<T, double> ? OZ2G_FP64 : OZ2G_FP32;
    oz2g_suggest s;
    detail::throw_status(oz2g_suggest_n_tight(prec, a.rows(), b.cols(), a.cols(), a.data(), a.cols(), b.data(),
                                              b.cols(), target, relative ? 1 : 0, OZ2G_HOST_PTRS, nullptr, &s));
    SuggestResult r;
    r.n = s.n;
    r.achievable = s.n > 0;
    r.bound_max = s.bound_max;
    return r;
}

// The same emulation tiled over several CUDA devices of this process
// (oz2g_gemm_multi): C is bit-identical to os_ii<T>; the result carries C,
// the subnormal flag and the table (no per-stage intermediates).
template <class T>
EmulationResult<T> os_ii_multi(const Matrix<T>& a, const Matrix<T>& b, int n, const std::vector<int>& devices) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
    require_dims(a.cols() == b.rows(), "os_ii inner dimension");
    const std::int64_t m = a.rows(), k = a.cols(), nn = b.cols();
    const int prec = std::is_same_v<T, double> ? OZ2G_FP64 : OZ2G_FP32;
    EmulationResult<T> r;
    r.C = Matrix<T>(m, nn);
    oz2g_diag diag;
    detail::throw_status(oz2g_gemm_multi(prec, m, nn, k, a.data(), k, b.data(), nn, r.C.data(), nn, n,
                                         OZ2G_HOST_PTRS, devices.data(), static_cast<int>(devices.size()), &diag));
    r.subnormal = diag.subnormal != 0;
    detail::throw_status(oz2g_table_for(n, prec, &r.table));
    return r;
}

// Tuning options of the library for this process (oz2g_set_option; names and
// values in oz2g.h).  std::invalid_argument for an unknown name or a value out
// of range.
inline void set_option(const std::string& name, long long value) {
    detail::throw_status(oz2g_set_option(name.c_str(), value));
}
inline long long get_option(const std::string& name) {
    long long v = 0;
    detail::throw_status(oz2g_get_option(name.c_str(), &v));
    return v;
}

}  // namespace oz2
