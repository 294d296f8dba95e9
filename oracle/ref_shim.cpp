// ref_shim.cpp — exports the GMP-free part of the REFERENCE hot path as a C
// ABI, compiled straight from the reference headers where they lie
// (-I/root/reference/proj/include; nothing is copied).  Builds
// oracle/_ref/liboz2_ref.so.  Test infrastructure only.
//
// What compiles without GMP/MPFR headers (absent in this image): matrix.hpp,
// parallel.hpp, int8gemm.hpp (the INT8 engine, the hottest loop of os_ii),
// prng.hpp and gen.hpp (the synthetic-input generator).  Everything that
// includes moduli.hpp/mp.hpp/dyadic.hpp needs <gmpxx.h>/<mpfr.h> and is
// unbuildable here; oracle/oz2_oracle.c restates those parts.
#include <oz2/gen.hpp>
#include <oz2/int8gemm.hpp>
#include <oz2/parallel.hpp>
#include <oz2/prng.hpp>

#include <cstring>
#include <exception>
#include <stdexcept>

extern "C" {

void ref_set_threads(int t) { oz2::worker_threads() = t < 1 ? 1 : t; }

int ref_gen_matrix_f64(long long rows, long long cols, double phi, unsigned long long seed, double* out) {
    try {
        const auto m = oz2::gen_matrix<double>(rows, cols, phi, seed);
        std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(rows * cols));
        return 0;
    } catch (const std::domain_error&) { return 2; } catch (...) { return 5; }
}

int ref_gen_matrix_f32(long long rows, long long cols, double phi, unsigned long long seed, float* out) {
    try {
        const auto m = oz2::gen_matrix<float>(rows, cols, phi, seed);
        std::memcpy(out, m.data(), sizeof(float) * static_cast<size_t>(rows * cols));
        return 0;
    } catch (const std::domain_error&) { return 2; } catch (...) { return 5; }
}

void ref_xoshiro_next(unsigned long long seed, long long count, unsigned long long* out) {
    oz2::Xoshiro256ss r(seed);
    for (long long i = 0; i < count; ++i) out[i] = r.next();
}

// int8gemm.hpp:17-34 on caller-owned row-major buffers.
int ref_gemm_i8_wrap(long long m, long long k, long long n, const signed char* a, const signed char* b, int* c) {
    try {
        oz2::MatrixI8 A(m, k), B(k, n);
        std::memcpy(A.data(), a, static_cast<size_t>(m * k));
        std::memcpy(B.data(), b, static_cast<size_t>(k * n));
        const oz2::MatrixI32 C = oz2::gemm_i8_wrap(A, B);
        std::memcpy(c, C.data(), sizeof(int) * static_cast<size_t>(m * n));
        return 0;
    } catch (const std::invalid_argument&) { return 1; }
    catch (const std::domain_error&) { return 2; } catch (...) { return 5; }
}

}  // extern "C"
