"""Seeded random cases against the oracle (a stand-in for compute-sanitizer,
which this pool does not allow): random shapes including degenerate ones,
both precisions, random N within each mode's range, random exponent spread,
host and device pointers, and strided device operands.  Each C is written into
a larger sentinel-filled buffer; a write outside the declared m x n window
fails the test, as does any difference from the oracle (bit-exact C, the same
exception and message on the error paths)."""
import os

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

pytestmark = pytest.mark.gpu

SENTINEL = -123.25
ORACLE_TO_OURS = {"OracleDomainError": oz.DomainError, "OracleRangeError": oz.RangeError,
                  "OracleLogicError": oz.LogicError, "OracleInvalidArgument": oz.InvalidArgument}


def _case(rng):
    shape_kind = rng.integers(0, 4)
    if shape_kind == 0:
        m, k, n = (int(x) for x in rng.integers(1, 9, size=3))
    elif shape_kind == 1:
        m, k, n = (int(x) for x in rng.integers(1, 300, size=3))
    elif shape_kind == 2:
        m, n = (int(x) for x in rng.integers(120, 520, size=2))
        k = int(rng.integers(1, 1100))
    else:
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        k = int(rng.integers(1000, 5000))
    dt = np.float64 if rng.random() < 0.7 else np.float32
    N = int(rng.integers(2, 50 if dt == np.float64 else 17))
    phi = float(rng.choice([0.0, 0.5, 2.0, 8.0]))
    return m, k, n, dt, N, phi


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_against_oracle(cuda, oracle, seed):
    import torch
    rng = np.random.default_rng(9000 + seed)
    m, k, n, dt, N, phi = _case(rng)
    A = oracle.gen_matrix(m, k, phi, 4000 + seed).astype(dt)
    B = oracle.gen_matrix(k, n, phi, 5000 + seed).astype(dt)
    try:
        ref = oracle.os_ii(A, B, N)
        ref_err = None
    except Exception as e:  # noqa: BLE001 - the device must raise the same
        ref, ref_err = None, e

    # host pointers, C written into a padded buffer through the C ABI view
    pad_r, pad_c = int(rng.integers(0, 3)), int(rng.integers(0, 5))
    big = np.full((m + pad_r, n + pad_c), SENTINEL, dtype=dt)
    out = big[:m, :n]
    use_out = pad_c == 0  # numpy slices with column padding are not row-major contiguous
    try:
        got = oz.os_ii(A, B, N, out=out if use_out else None)
        got_err = None
    except Exception as e:  # noqa: BLE001
        got, got_err = None, e
    if ref_err is not None:
        assert isinstance(got_err, ORACLE_TO_OURS[type(ref_err).__name__]), (got_err, ref_err)
        assert str(got_err) == str(ref_err)
        return
    assert got_err is None, got_err
    assert np.array_equal(got.C.view(np.uint8), ref.C.view(np.uint8))
    if use_out:
        assert np.all(big[m:, :] == SENTINEL)

    # device pointers with strided operands and a padded output
    lda, ldb, ldc = k + int(rng.integers(0, 9)), n + int(rng.integers(0, 9)), n + int(rng.integers(0, 9))
    tdt = torch.float64 if dt == np.float64 else torch.float32
    Ad = torch.full((m, lda), 7.0, dtype=tdt, device="cuda")
    Bd = torch.full((k, ldb), 7.0, dtype=tdt, device="cuda")
    Cd = torch.full((m + 2, ldc), SENTINEL, dtype=tdt, device="cuda")
    Ad[:, :k] = torch.from_numpy(A).cuda()
    Bd[:, :n] = torch.from_numpy(B).cuda()
    oz.os_ii(Ad[:, :k], Bd[:, :n], N, out=Cd[:m, :n])
    Ch = Cd.cpu().numpy()
    assert np.array_equal(np.ascontiguousarray(Ch[:m, :n]).view(np.uint8), ref.C.view(np.uint8))
    assert np.all(Ch[:m, n:] == SENTINEL) and np.all(Ch[m:, :] == SENTINEL)


@pytest.mark.parametrize("seed", range(int(os.environ.get("OZ2G_FUZZ_SEEDS", "8"))))
def test_fuzz_pipelined_host_path(cuda, oracle, seed):
    """Random shapes large enough for the pipelined host path (m >= 2048,
    n >= 256), random N, precision and exponent spread, under each
    speculation mode (OZ2G_SPEC 0 / 1 / 2): C bit-exact, the same exception
    and message on the error paths."""
    import os
    rng = np.random.default_rng(7100 + seed)
    m, n, k = int(rng.integers(2048, 3200)), int(rng.integers(256, 1600)), int(rng.integers(1, 130))
    dt = np.float64 if rng.random() < 0.7 else np.float32
    N = int(rng.integers(2, 21 if dt == np.float64 else 17))
    phi = float(rng.choice([0.0, 0.5, 2.0, 8.0]))
    A = oracle.gen_matrix(m, k, phi, 7200 + seed).astype(dt)
    B = oracle.gen_matrix(k, n, phi, 7300 + seed).astype(dt)
    try:
        ref, ref_err = oracle.os_ii(A, B, N), None
    except Exception as e:  # noqa: BLE001 - the device must raise the same
        ref, ref_err = None, e
    for mode in (0, 1, 2):
        try:
            with oz.options(spec=mode):
                got, got_err = oz.os_ii(A, B, N), None
        except Exception as e:  # noqa: BLE001
            got, got_err = None, e
        if ref_err is not None:
            assert isinstance(got_err, ORACLE_TO_OURS[type(ref_err).__name__]), (mode, got_err, ref_err)
            assert str(got_err) == str(ref_err), mode
            continue
        assert got_err is None, (mode, got_err)
        assert np.array_equal(got.C.view(np.uint8), ref.C.view(np.uint8)), (mode, m, k, n, N, phi, dt)
