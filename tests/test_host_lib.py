"""CPU-side checks of the native library (no GPU needed):

* liboz2g.so loads and exports every entry point include/oz2g.h declares;
* the natively built constant tables (tables.cpp) equal the oracle's exact
  restatement of build_table for every N in [2, 49] and both modes;
* the device step table for the scaling exponents reproduces the oracle's
  direct evaluation of scaling.hpp:171-180 around every threshold and on a
  random sample of clearance maxima;
* argument validation happens before any device work (reference error classes).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2602_02549_b200 as oz
from paper_2602_02549_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    L = oz.load_library()
    header = open(os.path.join(ROOT, "include", "oz2g.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|uint64_t|const char \*)\s*\**\s*(oz2g_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name


def test_version():
    assert oz.load_library().oz2g_version() == 4


@pytest.mark.parametrize("mode", [oz.F32, oz.F64])
def test_tables_match_oracle(mode):
    from oracle import moduli as M
    for n in range(2, 50):
        t = oz.table_for(n, mode)
        o = M.build_table(n, mode)
        assert t.p == o["p"] and t.q == o["q"] and t.P == o["P"] and t.rho == o["rho"]
        assert t.P1 == o["P1"] and t.P2 == o["P2"] and t.P_inv == o["P_inv"]
        assert t.beta == o["beta"] and t.s1 == o["s1"] and t.s2 == o["s2"]
        assert t.P_prime == o["P_prime"]


def test_fp32_ceiling():
    assert oz.fp32_safe_moduli_max() == 16


def test_table_for_domain_error():
    for bad in (1, 50, 0, -3):
        with pytest.raises(oz.DomainError):
            oz.table_for(bad)


@pytest.mark.parametrize("n", [2, 6, 8, 14, 16, 20, 33, 49])
def test_step_table_reproduces_shift(oracle, n):
    t = oz.table_for(n)
    thr = t.thresholds

    def shift_tab(c):
        return t.shift0 - sum(1 for x in thr if c >= x)

    probes = {0, 1, 2, 3, (1 << 29) - 1, 1 << 29}
    for x in thr:
        probes.update({x - 1, x, x + 1})
    rng = np.random.default_rng(n)
    probes.update(int(v) for v in rng.integers(0, 1 << 29, 300))
    probes.update(int(2 ** e) for e in np.linspace(0, 29, 200))
    for c in sorted(probes):
        s_or, _ = oracle.shift_of_cmax(c, n)
        assert shift_tab(c) == s_or, (n, c)
        assert oz.load_library().oz2g_shift_of_cmax(n, c) == s_or


def test_survey_thresholds():
    import json
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "shift_thresholds.json")))
    for n, (s0, thr) in ((int(k), v) for k, v in gold["shift0_and_thresholds"].items()):
        t = oz.table_for(n)
        assert t.shift0 == s0 and t.thresholds == thr


def test_validation_before_device_work():
    # k > 2^17: domain error (emulate.hpp:59), raised before touching the device
    A = np.ones((1, (1 << 17) + 1))
    B = np.ones(((1 << 17) + 1, 1))
    with pytest.raises(oz.DomainError, match="k exceeds"):
        oz.os_ii(A, B, 5)
    with pytest.raises(oz.InvalidArgument):
        oz.os_ii(np.ones((2, 3)), np.ones((4, 2)), 5)
    with pytest.raises(oz.DomainError, match="N out of"):
        oz.os_ii(np.ones((2, 3)), np.ones((3, 2)), 50)
    with pytest.raises(oz.DomainError, match="zero row"):  # k == 0: every row is zero
        oz.os_ii(np.ones((2, 0)), np.ones((0, 2)), 5)
    with pytest.raises(TypeError):
        oz.os_ii(np.ones((2, 3), dtype=np.float32), np.ones((3, 2)), 5)
