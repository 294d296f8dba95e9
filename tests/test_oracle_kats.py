"""The CPU oracle pinned against the reference's own known-answer tests.

Each test cites the reference test it ports (/root/reference/proj/tests/).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import moduli as M


# ---------------------------------------------------------------- moduli
def test_fixed_moduli_list():  # test_moduli.cpp:12-23
    assert len(M.K_MODULI) == 49
    assert M.K_MODULI[0] == 256 and M.K_MODULI[1] == 255 and M.K_MODULI[4] == 247 and M.K_MODULI[48] == 29
    for i, a in enumerate(M.K_MODULI):
        assert a <= 256
        for b in M.K_MODULI[i + 1:]:
            assert math.gcd(a, b) == 1


def test_mod_inverse_examples():  # test_moduli.cpp:25-30
    assert M.mod_inverse(255, 256) == 255
    assert M.mod_inverse(256, 255) == 1
    assert M.mod_inverse(1, 97) == 1
    with pytest.raises(ValueError):
        M.mod_inverse(12, 256)


def test_split_upper_bits():  # test_moduli.cpp:32-43
    assert M.split_upper_bits(0b10110110, 4) == (float(0b10110000), float(0b0110))
    assert M.split_upper_bits((1 << 53) - 1, 53) == (2.0 ** 53 - 1, 0.0)
    assert M.split_upper_bits((1 << 60) + 1, 30) == (2.0 ** 60, 1.0)
    with pytest.raises(ValueError):
        M.split_upper_bits(5, 0)


def test_n2_table():  # test_moduli.cpp:45-62
    t = M.build_table(2, M.F64)
    assert t["p"] == [256, 255] and t["q"] == [255, 1]
    assert t["P"] == 65280 and t["rho"] == 255
    assert t["r"] == [65025, 256]
    assert t["P1"] == 65280.0 and t["P2"] == 0.0
    assert math.floor(t["P_prime"]) == 7
    for l in range(2):
        assert 0 < t["q"][l] < t["p"][l]
        assert t["r"][l] % t["p"][l] == 1


@pytest.mark.parametrize("mode", [M.F32, M.F64])
def test_inverse_property_all_n(mode):  # test_moduli.cpp:64-81
    for n in range(2, 50):
        t = M.build_table(n, mode)
        prod = 1
        for l in range(n):
            assert t["r"][l] % t["p"][l] == 1
            assert t["q"][l] < t["p"][l]
            prod *= t["p"][l]
        assert t["rho"] == sum(p // 2 for p in t["p"])
        assert t["P"] == prod
        assert t["P_prime"] < 200.0


def test_double_double_P():  # test_moduli.cpp:83-93
    for n in (2, 5, 10, 20, 30, 49):
        t = M.build_table(n, M.F64)
        err = abs(Fraction(t["P"]) - (Fraction(t["P1"]) + Fraction(t["P2"])))
        assert err <= Fraction(1, 1 << 106) * t["P"] / 2
        t32 = M.build_table(n, M.F32)
        assert t32["P2"] == 0.0 and all(s == 0.0 for s in t32["s2"])


def test_s1_s2_invariants():  # test_moduli.cpp:95-124
    for n in (2, 5, 13, 20, 34, 49):
        t = M.build_table(n, M.F64)
        rmax = max(t["r"])
        ufp_bits = rmax.bit_length() - 1
        clr = M.ceil_log2_long(t["rho"])
        quantum_exp = clr - 53 + ufp_bits + 1
        for l in range(n):
            s1 = int(t["s1"][l])
            assert Fraction(t["s1"][l]) == s1
            assert 0 <= s1 < (1 << (ufp_bits + 1))
            if quantum_exp > 0:
                assert s1 % (1 << quantum_exp) == 0
            rem = t["r"][l] - s1
            assert rem >= 0
            assert Fraction(rem) < Fraction(1 << (1 + clr), 1 << 53) * t["P"]
            recon = abs(Fraction(t["r"][l]) - (Fraction(s1) + Fraction(t["s2"][l])))
            assert recon <= (1 << max(quantum_exp, 1))


def test_fp32_s1_nearest():  # test_moduli.cpp:126-133
    for n in (2, 10, 16):
        t = M.build_table(n, M.F32)
        for l in range(n):
            assert t["s1"][l] == float(t["r"][l])


def test_p_inv_correctly_rounded():  # test_moduli.cpp:135-142
    for n in (2, 7, 49):
        t = M.build_table(n, M.F64)
        diff = abs(Fraction(1, t["P"]) - Fraction(t["P_inv"]))
        ufp = Fraction(2) ** math.floor(math.log2(t["P_inv"]))
        assert diff <= ufp / (1 << 53)


def test_crt_reconstruction_identity():  # test_moduli.cpp:144-150 (selfcheck.hpp:327-343)
    rng = np.random.default_rng(77)
    for n in range(2, 50):
        t = M.build_table(n, M.F64)
        for _ in range(20):
            x = int(rng.integers(-2 ** 62, 2 ** 62)) * int(rng.integers(1, 2 ** 40)) % t["P"]
            res = [x % p for p in t["p"]]
            rec = sum(r_l * w for r_l, w in zip(t["r"], res)) % t["P"]
            assert rec == x % t["P"]


def test_table_rejects_out_of_range():  # test_moduli.cpp:152-155
    for bad in (1, 50):
        with pytest.raises(ValueError):
            M.build_table(bad, M.F64)


def test_fp32_ceiling():  # test_moduli.cpp:157-164, README.md:131-141
    cap = M.fp32_safe_moduli_max()
    assert cap == 16
    limit = ((1 << 24) - 1) << 105
    assert M.build_table(cap, M.F32)["P"] <= limit
    assert M.build_table(cap + 1, M.F32)["P"] > limit


def test_scaling_coeff():  # test_scaling.cpp:84-86
    assert M.scaling_coeff_fp32() == float.fromhex("-0x1.000006p-1")


def test_p_prime_floors_survey():
    for n, fl in {2: 7, 6: 23, 7: 27, 8: 31, 14: 54, 16: 62, 17: 65}.items():
        assert math.floor(M.build_table(n, M.F64)["P_prime"]) == fl


# ---------------------------------------------------------------- softfp
def test_round_nearest_even(oracle):  # test_softfp.cpp:14-22
    R = oracle.round_nearest_even
    assert R(1.75) == 2.0 and R(0.5) == 0.0 and R(-2.5) == -2.0 and R(2.5) == 2.0
    assert R(3.5) == 4.0 and R(-0.49) == 0.0 and R(2.0 ** 53) == 2.0 ** 53


def test_signed_mod(oracle):  # test_softfp.cpp:30-43
    S = oracle.signed_mod
    assert S(300, 256) == 44 and S(7, 4) == -1 and S(128, 256) == 128 and S(-7, 4) == 1 and S(384, 256) == -128
    rng = np.random.default_rng(1)
    for _ in range(2000):
        x = int(rng.integers(-2 ** 40, 2 ** 40))
        p = int(rng.integers(2, 300))
        r = S(x, p)
        assert (x - r) % p == 0 and abs(r) <= p // 2


def test_fp32_round_up(oracle):  # test_softfp.cpp:115-120
    assert oracle.lib().ora_fp32_round_up(0) == 0.0
    assert oracle.lib().ora_fp32_round_up((1 << 24) + 1) == float.fromhex("0x1.000002p24")
    assert oracle.lib().ora_fp32_round_up(1 << 24) == 2.0 ** 24
    assert oracle.lib().ora_fp32_round_up((1 << 29) - 1) >= (1 << 29) - 1


def test_log2f_anchors(oracle):  # test_softfp.cpp:100-109
    L = oracle.lib().ora_log2_fp32
    assert L(1.0) == 0.0 and L(1024.0) == 10.0
    import mpmath
    mpmath.mp.prec = 96
    expect = float(np.float32(float(mpmath.log(3, 2))))
    assert L(3.0) == expect


def test_fma_fp32_down_single_rounding(oracle):  # test_softfp.cpp:286-300 (directed variant)
    F = oracle.lib().ora_fma_fp32_down
    rng = np.random.default_rng(3)
    for _ in range(5000):
        a, b, c = (float(np.float32(x)) for x in rng.standard_normal(3) * rng.choice([1e-3, 1.0, 1e3], 3))
        exact = Fraction(a) * Fraction(b) + Fraction(c)
        got = F(a, b, c)
        assert Fraction(got) <= exact
        assert Fraction(float(np.nextafter(np.float32(got), np.float32(np.inf)))) > exact


# ---------------------------------------------------------------- scaling
def test_pre_exponents_and_ceil(oracle):  # test_scaling.cpp:13-40
    A = np.array([[1.0, -0.25], [0.3, 0.1], [2.0 ** 10, 3.0]])
    r = oracle.os_ii(A, np.ones((2, 1)), 5, keep_intermediates=True)
    assert r.inter["mu_prime"].tolist() == [5, 7, -5]
    assert oracle.ceil_abs_scaled(-0.3, 5) == 10
    assert oracle.ceil_abs_scaled(0.0, 5) == 0
    assert oracle.ceil_abs_scaled(1.0, 5) == 32


def test_zero_row_and_col_rejected(oracle):  # test_scaling.cpp:21-28, test_emulate.cpp:113-120
    z = np.zeros((2, 2)); z[0, 0] = 1.0
    with pytest.raises(oracle.OracleDomainError):
        oracle.os_ii(z, np.ones((2, 2)), 5)
    zc = np.zeros((2, 2)); zc[0, 0] = 1.0; zc[1, 0] = 2.0
    with pytest.raises(oracle.OracleDomainError):
        oracle.os_ii(np.ones((2, 2)), zc, 5)


def test_subnormal_ceil(oracle):  # test_scaling.cpp:60-71
    assert oracle.ceil_abs_scaled(2.0 ** -1069, 5 - 1000) == 1
    assert oracle.ceil_abs_scaled(2.0 ** 1000, 5 - 1000) == 32


def test_row_peaks_in_range(oracle):  # test_scaling.cpp:42-58
    for it in range(50):
        A = oracle.gen_matrix(4, 8, 2.0, 1000 + it)
        r = oracle.os_ii(A, np.ones((8, 1)), 5, keep_intermediates=True)
        for i in range(4):
            ab = [oracle.ceil_abs_scaled(A[i, h], int(r.inter["mu_prime"][i])) for h in range(8)]
            assert all(1 <= v <= 64 for v in ab) and max(ab) >= 32


def test_scaling_exponent_kats(oracle):  # test_scaling.cpp:88-105
    s, e = oracle.shift_of_cmax(1, 2)       # Dbar max 1 -> e = 0 -> mu - mu' = floor(P') = 7
    assert e == 0.0 and s == 7
    s0, e0 = oracle.shift_of_cmax(0, 2)     # zero row clamped to 1
    assert e0 == 0.0 and s0 == 7
    _, e4 = oracle.shift_of_cmax(4, 2)
    assert e4 == 2.0


def test_truncation(oracle):  # test_scaling.cpp:107-113
    A = np.array([[1.75, -1.75, 0.5]])
    r = oracle.os_ii(A, np.ones((3, 1)), 2, keep_intermediates=True)
    mu = int(r.inter["mu"][0])
    ap = r.inter["Aprime"][0]
    assert ap[0] == math.trunc(1.75 * 2.0 ** mu) and ap[1] == -ap[0]


import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SURVEY_THRESHOLDS = {int(k): (v[0], v[1]) for k, v in
                     json.load(open(os.path.join(GOLDEN, "shift_thresholds.json")))["shift0_and_thresholds"].items()}


@pytest.mark.parametrize("n", sorted(SURVEY_THRESHOLDS))
def test_shift_step_function_matches_survey(oracle, n):
    s0, thr = SURVEY_THRESHOLDS[n]
    assert oracle.shift_of_cmax(1, n)[0] == s0
    for j, t in enumerate(thr):
        assert oracle.shift_of_cmax(t, n)[0] == s0 - j - 1
        assert oracle.shift_of_cmax(t - 1, n)[0] == s0 - j


def test_log2f_monotone_exhaustive(oracle):
    """Every value Dbar can take (RU32 of integers in [1, 2^29]): log2f is
    monotone, so shift(c) is a step function and the device threshold table
    is exact."""
    assert oracle.lib().ora_log2f_monotone_violations() == 0


# ---------------------------------------------------------------- crt
def test_residue_kats(oracle):  # test_crt.cpp:12-28
    big = 3 << 60
    r = big % 251
    expect = r - 251 if 2 * r > 251 else r
    assert oracle.residue_of(3.0 * 2.0 ** 60, 251) == expect
    assert oracle.residue_of(-7.0, 4) == 1
    assert oracle.residue_of(128.0, 256) == -128
    with pytest.raises(oracle.OracleDomainError):
        oracle.residue_of(0.5, 7)


def test_residues_random_huge(oracle):  # test_crt.cpp:30-47
    rng = np.random.default_rng(0xfeed)
    for _ in range(500):
        mant = int(rng.integers(0, 2 ** 53))
        e = int(rng.integers(0, 120))
        neg = bool(rng.integers(0, 2))
        v = math.ldexp(-mant if neg else mant, e)
        if v == 0:
            continue
        big = int(Fraction(v))
        for p in (256, 255, 251, 97, 29, 4, 3, 2):
            r = oracle.residue_of(v, p)
            assert (big - r) % p == 0 and abs(r) <= p // 2


def test_int8_engine_kats(oracle):  # test_int8gemm.cpp:11-26, test_crt.cpp:58-65
    assert oracle.gemm_i8_wrap(np.full((1, 1), 127), np.full((1, 1), 127))[0, 0] == 16129
    K = 1 << 17
    c = oracle.gemm_i8_wrap(np.full((1, K), -128), np.full((K, 1), -128))
    assert c[0, 0] == -(2 ** 31)
    assert oracle.signed_mod(int(c[0, 0]), 256) in (0,)
    c = oracle.gemm_i8_wrap(np.full((1, K), 64), np.full((K, 1), 64))
    assert c[0, 0] == 1 << 29


def test_accumulate_exact_fp64(oracle):  # test_crt.cpp:67-92 (Lemma 2: C1 exact in fp64 mode)
    A = oracle.gen_matrix(3, 12, 1.5, 0x1111)
    B = oracle.gen_matrix(12, 3, 1.5, 0x2222)
    for n in (5, 14, 30):
        r = oracle.os_ii(A, B, n, keep_intermediates=True)
        t = M.build_table(n, M.F64)
        W = r.inter["W"]
        for i in range(3):
            for j in range(3):
                exact = sum(Fraction(t["s1"][l]) * int(W[l, i, j]) for l in range(n))
                assert Fraction(r.inter["C1"][i, j]) == exact


def test_q_kat(oracle):  # test_crt.cpp:94-109  W = (1, 0): C1 = 65025, Q = 1
    t = M.build_table(2, M.F64)
    c1 = t["s1"][0] * 1
    assert c1 == 65025.0
    assert oracle.round_nearest_even(t["P_inv"] * c1) == 1.0


def test_crt_identity_end_to_end(oracle):  # test_crt.cpp:147-167
    for n in (2, 8, 20):
        A = oracle.gen_matrix(3, 12, 1.5, 0x1111 + n)
        B = oracle.gen_matrix(12, 3, 1.5, 0x2222 + n)
        r = oracle.os_ii(A, B, n, keep_intermediates=True)
        t = M.build_table(n, M.F64)
        Ap = [[int(x) for x in row] for row in r.inter["Aprime"]]
        Bp = [[int(x) for x in row] for row in r.inter["Bprime"]]
        for i in range(3):
            for j in range(3):
                ab = sum(Ap[i][h] * Bp[h][j] for h in range(12))
                cex = sum(t["r"][l] * int(r.inter["W"][l, i, j]) for l in range(n))
                modp = cex % t["P"]
                if 2 * modp > t["P"]:
                    modp -= t["P"]
                assert modp == ab
                assert abs(r.inter["Q"][i, j]) <= t["rho"] + 0.5
                assert 2 * sum(abs(Ap[i][h] * Bp[h][j]) for h in range(12)) < t["P"]


# ---------------------------------------------------------------- emulate
def test_unit_product_trace(oracle):  # test_emulate.cpp:13-37
    one = np.ones((1, 1))
    r = oracle.os_ii(one, one, 2, keep_intermediates=True)
    assert r.C[0, 0] == 1.0
    assert r.inter["mu"][0] == 7 and r.inter["nu"][0] == 7
    assert r.inter["Aprime"][0, 0] == 128.0 and r.inter["Bprime"][0, 0] == 128.0
    assert r.inter["W"][:, 0, 0].tolist() == [0, 64]
    assert r.inter["C1"][0, 0] == 16384.0 and r.inter["Q"][0, 0] == 0.0 and r.inter["Cpp64"][0, 0] == 16384.0
    assert oracle.os_ii(one.astype(np.float32), one.astype(np.float32), 2).C[0, 0] == 1.0
    for n in (10, 30, 49):
        assert abs(oracle.os_ii(one, one, n).C[0, 0] - 1.0) <= 2.0 ** -40
    for n in (10, 16):
        assert abs(float(oracle.os_ii(one.astype(np.float32), one.astype(np.float32), n).C[0, 0]) - 1.0) <= 2.0 ** -18


def test_fp32_range_error_beyond_ceiling(oracle):  # test_emulate.cpp:67-73, test_crt.cpp:118-125
    a = oracle.gen_matrix(3, 8, 0.5, 0xcc, np.float32)
    b = oracle.gen_matrix(8, 3, 0.5, 0xdd, np.float32)
    with pytest.raises(oracle.OracleRangeError):
        oracle.os_ii(a, b, M.fp32_safe_moduli_max() + 1)


def test_deterministic_across_threads(oracle):  # test_emulate.cpp:75-87
    a = oracle.gen_matrix(9, 40, 2.0, 0xee)
    b = oracle.gen_matrix(40, 9, 2.0, 0xff)
    oracle.set_threads(1)
    r1 = oracle.os_ii(a, b, 25).C
    oracle.set_threads(8)
    r8 = oracle.os_ii(a, b, 25).C
    oracle.set_threads(1)
    assert r1.tobytes() == r8.tobytes()


def test_pow2_inverse_exact(oracle):  # test_emulate.cpp:89-100
    a = oracle.gen_matrix(4, 12, 1.0, 0x1234)
    b = oracle.gen_matrix(12, 4, 1.0, 0x4321)
    r = oracle.os_ii(a, b, 12, keep_intermediates=True)
    assert not r.subnormal
    for i in range(4):
        for j in range(4):
            back = math.ldexp(math.ldexp(r.C[i, j], int(r.inter["mu"][i])), int(r.inter["nu"][j]))
            assert back == r.inter["Cpp64"][i, j]


def test_preconditions(oracle):  # test_emulate.cpp:113-120
    a = np.zeros((2, 3)); a[0] = 1.0
    b = np.ones((3, 2))
    with pytest.raises(oracle.OracleDomainError):
        oracle.os_ii(a, b, 5)
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.os_ii(a, np.ones((4, 2)), 5)


def test_error_vs_native_small(oracle):  # acceptance.cpp:123-124 style saturation check
    a = oracle.gen_matrix(16, 64, 0.5, 5)
    b = oracle.gen_matrix(64, 16, 0.5, 6)
    exact = [[sum(Fraction(a[i, h]) * Fraction(b[h, j]) for h in range(64)) for j in range(16)] for i in range(16)]
    r = oracle.os_ii(a, b, 20)
    err = max(abs(Fraction(r.C[i, j]) - exact[i][j]) for i in range(16) for j in range(16))
    native = a @ b
    err_nat = max(abs(Fraction(native[i, j]) - exact[i][j]) for i in range(16) for j in range(16))
    assert err <= 100 * err_nat


# ---------------------------------------------------------------- generator (reference stream)
def test_generator_matches_reference_build(oracle):
    """oracle/_ref is the reference's own gen.hpp/prng.hpp compiled in place."""
    R = oracle.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built (reference headers absent)")
    for phi, dt, fn in ((0.0, np.float64, R.ref_gen_matrix_f64), (2.0, np.float64, R.ref_gen_matrix_f64),
                        (8.0, np.float32, R.ref_gen_matrix_f32)):
        ours = oracle.gen_matrix(13, 17, phi, 0x77, dt)
        ref = np.empty((13, 17), dtype=dt)
        assert fn(13, 17, phi, 0x77, ref.ctypes.data) == 0
        assert ours.tobytes() == ref.tobytes()


def test_int8_engine_matches_reference_build(oracle):
    R = oracle.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built (reference headers absent)")
    rng = np.random.default_rng(5)
    a = rng.integers(-128, 128, (19, 300), dtype=np.int8)
    b = rng.integers(-128, 128, (300, 23), dtype=np.int8)
    ref = np.empty((19, 23), dtype=np.int32)
    assert R.ref_gemm_i8_wrap(19, 300, 23, a.ctypes.data, b.ctypes.data, ref.ctypes.data) == 0
    assert np.array_equal(oracle.gemm_i8_wrap(a, b), ref)


def test_oracle_reproduces_reference_golden(oracle):
    """Committed fixtures produced by the reference's own gen.hpp / int8gemm.hpp
    (tests/golden/make_golden.py); valid where /root/reference is absent."""
    g = np.load(os.path.join(GOLDEN, "ref_gen_gemm.npz"))
    cases = json.load(open(os.path.join(GOLDEN, "gen_cases.json")))
    for idx, (r, c, phi, seed, dt) in enumerate(cases):
        ours = oracle.gen_matrix(r, c, phi, seed, np.float64 if dt == "f64" else np.float32)
        assert ours.tobytes() == g[f"gen{idx}"].tobytes()
    for idx in range(3):
        assert np.array_equal(oracle.gemm_i8_wrap(g[f"gemm{idx}_a"], g[f"gemm{idx}_b"]), g[f"gemm{idx}_c"])


def test_sampled_pieces_equal_full_oracle(oracle):
    """The sampled full-size checkers reproduce the full oracle exactly."""
    for phi, dt in ((2.0, np.float64), (0.5, np.float32)):
        A = oracle.gen_matrix(40, 50, phi, 1, dt)
        B = oracle.gen_matrix(50, 30, phi, 2, dt)
        r = oracle.os_ii(A, B, 16, keep_intermediates=True)
        A64, B64 = A.astype(np.float64), B.astype(np.float64)
        mup = oracle.pre_exponents(A64, False)
        nup = oracle.pre_exponents(B64, True)
        assert np.array_equal(mup, r.inter["mu_prime"]) and np.array_equal(nup, r.inter["nu_prime"])
        ab, bb = oracle.ceil_scale(A64, mup, False), oracle.ceil_scale(B64, nup, True)
        assert np.array_equal(oracle.cbar_row_max(ab, bb, np.arange(40)), r.inter["cmax_row"])
        assert np.array_equal(oracle.cbar_col_max(ab, bb, np.arange(30)), r.inter["cmax_col"])
        ri, cj = np.repeat(np.arange(40), 30), np.tile(np.arange(30), 40)
        e = oracle.entries(A64, B64, 16, r.inter["mu"], r.inter["nu"], ri, cj, prec=1 if dt == np.float64 else 0)
        assert e.reshape(40, 30).tobytes() == r.C.tobytes()
