"""Harness and CLI: reference stream, matrix text
format, CLI subcommands, error-vs-bound sweep."""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_02549_b200 as oz
from paper_2602_02549_b200 import experiment as X
from paper_2602_02549_b200 import matrix_io as MIO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _c_hex(v: float) -> str:
    libc = ctypes.CDLL(None)
    buf = ctypes.create_string_buffer(64)
    libc.snprintf(buf, 64, b"%a", ctypes.c_double(v))
    return buf.value.decode()


def test_hexfloat_matches_c_printf():
    vals = [0.0, -0.0, 1.0, -1.5, 0.1, 3.0 * 2 ** 60, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
            float.fromhex("0x1.000006p-1"), -7.25e-300, float("inf"), -float("inf")]
    rng = np.random.default_rng(0)
    vals += list(rng.standard_normal(200) * 10.0 ** rng.integers(-300, 300, 200))
    for v in vals:
        assert MIO.hexfloat(v) == _c_hex(v), v


def test_matrix_file_roundtrip(tmp_path):
    for dt in (np.float64, np.float32):
        m = (np.random.default_rng(1).standard_normal((5, 7)) * 1e-3).astype(dt)
        p = str(tmp_path / "m.mat")
        MIO.write_matrix(p, m)
        back = MIO.read_matrix(p)
        assert back.dtype == dt and back.tobytes() == m.tobytes()
        head = open(p).readline().split()
        assert head == ["5", "7", "fp64" if dt == np.float64 else "fp32"]


def test_library_stream_matches_reference_golden():
    g = np.load(os.path.join(GOLDEN, "ref_gen_gemm.npz"))
    cases = json.load(open(os.path.join(GOLDEN, "gen_cases.json")))
    for idx, (r, c, phi, seed, dt) in enumerate(cases):
        ours = X.gen_matrix(r, c, phi, seed, oz.F64 if dt == "f64" else oz.F32)
        assert ours.tobytes() == g[f"gen{idx}"].tobytes()


def test_derive_seed_matches_oracle(oracle):
    for s, t, r in [(1, 0, 0), (1, 0, 1), (12345, 7, 1), (2 ** 63 + 5, 3, 0)]:
        assert X.derive_seed(s, t, r) == oracle.derive_seed(s, t, r)


def test_validate_config():
    with pytest.raises(oz.DomainError):
        X.validate_config(X.ExperimentConfig(n_list=[]))
    with pytest.raises(oz.DomainError, match="fp32-safe"):
        X.validate_config(X.ExperimentConfig(mode=oz.F32, n_list=[17]))
    with pytest.raises(oz.DomainError):
        X.validate_config(X.ExperimentConfig(k=(1 << 17) + 1, n_list=[5]))


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2602_02549_b200.cli", *args], capture_output=True,
                          text=True, cwd=ROOT, timeout=600)


def test_cli_table_n2():
    out = _cli("table", "--n", "2", "--mode", "fp64")
    assert out.returncode == 0
    lines = out.stdout.splitlines()
    assert lines[0].startswith("P=65280,rho=255,P1=0x1.fe0000p+15".replace("0x1.fe0000p+15", "0x1.fep+15"))
    assert lines[1] == "ell,p,q,beta,s1,s2"
    assert lines[2].startswith("1,256,255,") and lines[3].startswith("2,255,1,")


def test_cli_errors_exit_2():
    assert _cli("table", "--n", "50", "--mode", "fp64").returncode == 2
    assert _cli("table", "--n", "5", "--mode", "fp16").returncode == 2


@pytest.mark.gpu
def test_cli_emulate_bounds_suggest(tmp_path, cuda, oracle):
    A = oracle.gen_matrix(12, 40, 1.0, 5)
    B = oracle.gen_matrix(40, 9, 1.0, 6)
    pa, pb, pc = str(tmp_path / "A.mat"), str(tmp_path / "B.mat"), str(tmp_path / "C.mat")
    MIO.write_matrix(pa, A)
    MIO.write_matrix(pb, B)
    assert _cli("emulate", "--a", pa, "--b", pb, "--n", "20", "--mode", "fp64", "--out", pc).returncode == 0
    assert MIO.read_matrix(pc).tobytes() == oracle.os_ii(A, B, 20).C.tobytes()
    r = _cli("bounds", "--a", pa, "--b", pb, "--n", "20", "--mode", "fp64", "--tight")
    assert r.returncode == 0 and r.stdout.startswith("bound=tight n=20 max=0x")
    r = _cli("suggest-n", "--a", pa, "--b", pb, "--target", "1e-10", "--mode", "fp64")
    assert r.returncode == 0 and r.stdout.startswith("n="), r.stdout + r.stderr
    # the truncation terms of the cheap bound do not shrink with N: ~3e-13 here
    r = _cli("suggest-n", "--a", pa, "--b", pb, "--target", "1e-14", "--mode", "fp64")
    assert r.returncode == 1 and r.stdout.startswith("not achievable"), r.stdout + r.stderr
    assert _cli("emulate", "--a", pa, "--b", pb, "--n", "20", "--mode", "fp32", "--out", pc).returncode == 2
    assert _cli("selftest").returncode == 0


@pytest.mark.gpu
def test_experiment_sweep(tmp_path, cuda):
    out = str(tmp_path / "sweep.csv")
    r = _cli("experiment", "--m", "16", "--n", "16", "--k", "256", "--phi", "0.5", "2", "--mode", "fp64",
             "--n-list", "4", "8", "14", "20", "--out", out)
    assert r.returncode == 0, r.stderr
    for phi in ("0.5", "2"):
        lines = open(str(tmp_path / f"sweep.phi{phi}.csv")).read().splitlines()
        assert lines[0] == "n,est_max,est_min,est2_max,est2_min,err_max,err_min,err_native_max,err_max_dec"
        assert len(lines) == 5
        for ln in lines[1:]:
            f = ln.split(",")
            est_max, est_min, est2_max = (float.fromhex(v) for v in f[1:4])
            err_max, err_min = float.fromhex(f[5]), float.fromhex(f[6])
            assert err_max <= est_max <= est2_max and err_min <= est_min


@pytest.mark.gpu
def test_experiment_error_matches_exact(cuda, oracle):
    """err_* of the GPU sweep equal the exact errors (GMP semantics of
    error_matrix, oracle.hpp:164-172) up to the fp64 rounding of the report."""
    from fractions import Fraction
    from oracle import bounds as OB
    cfg = X.ExperimentConfig(m=8, n=7, k=64, phi=1.0, n_list=[6, 12], seed=3)
    rows = X.run_experiment(cfg)
    a = oracle.gen_matrix(8, 64, 1.0, oracle.derive_seed(3, 0, 0))
    b = oracle.gen_matrix(64, 7, 1.0, oracle.derive_seed(3, 0, 1))
    exact = OB.exact_product(a, b)
    for row in rows:
        c = oracle.os_ii(a, b, row.n).C
        errs = [abs(Fraction(float(c[i, j])) - exact[i][j]) for i in range(8) for j in range(7)]
        emax = float(max(errs))
        assert abs(row.err_max - emax) <= 2.0 ** -50 * emax + 1e-300
