"""Error behaviour of the device pipeline against the oracle (emulate.hpp:54-88
and the checks it reaches: scaling.hpp:33-52 / :86-107 zero rows and columns,
non-finite entries, emulate.hpp:30-46 inverse-scaling overflow).  The device
raises the reference's exception class with the reference's message, for the
device-pointer path and for the pipelined host-pointer path (where the row
exponents and A residues of early chunks run before the last chunk lands)."""

import numpy as np
import pytest

import paper_2602_02549_b200 as oz

ORACLE_TO_OURS = {"OracleDomainError": oz.DomainError, "OracleRangeError": oz.RangeError,
                  "OracleLogicError": oz.LogicError}


def _cases(oracle, m, k, n):
    A = oracle.gen_matrix(m, k, 1.0, 71)
    B = oracle.gen_matrix(k, n, 1.0, 72)
    out = {}
    a = A.copy(); a[m - 7, :] = 0.0
    out["zero row (last chunk)"] = (a, B)
    a = A.copy(); a[3, :] = 0.0
    out["zero row (first chunk)"] = (a, B)
    b = B.copy(); b[:, n - 2] = 0.0
    out["zero column"] = (A, b)
    a = A.copy(); a[m // 2, 5] = np.nan
    out["nan in A"] = (a, B)
    b = B.copy(); b[1, 3] = -np.inf
    out["inf in B"] = (A, b)
    out["inverse-scaling overflow"] = (A * 1e200, B * 1e200)
    a = A.copy(); a[m - 7, :] = 0.0
    b = B.copy(); b[:, 1] = 0.0
    out["zero row and column: the row is reported"] = (a, b)
    # the first failing row / column decides the message, whatever its kind
    # (scaling.hpp:33-52 and :86-107 scan in order)
    a = A.copy(); a[3, :] = 0.0; a[m - 7, 5] = np.nan
    out["zero row before a nan row"] = (a, B)
    a = A.copy(); a[2, 1] = np.nan; a[m - 7, :] = 0.0
    out["nan row before a zero row"] = (a, B)
    b = B.copy(); b[:, 1] = 0.0; b[2, n - 2] = np.inf
    out["zero column before an inf column"] = (A, b)
    b = B.copy(); b[0, 1] = np.inf; b[:, n - 2] = 0.0
    out["inf column before a zero column"] = (A, b)
    return out


def _expect(oracle, a, b, nmod):
    try:
        oracle.os_ii(a, b, nmod)
    except Exception as e:  # noqa: BLE001 - the oracle's class picks ours
        return ORACLE_TO_OURS[type(e).__name__], str(e)
    return None, None


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n", [(64, 48, 40), (2560, 64, 300), (2560, 64, 1100)])
def test_errors_match_oracle(cuda, oracle, m, k, n):
    import torch
    for name, (a, b) in _cases(oracle, m, k, n).items():
        cls, msg = _expect(oracle, a, b, 14)
        assert cls is not None, name
        # host pointers (pipelined for the large shapes, under every speculation mode)
        for mode in ((0, 1, 2) if m >= 2048 else (-1,)):
            with oz.options(spec=mode), pytest.raises(cls) as ei:
                oz.os_ii(a, b, 14)
            assert str(ei.value) == msg, (name, mode, str(ei.value), msg)
        # device pointers
        with pytest.raises(cls) as ei:
            oz.os_ii(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 14)
        assert str(ei.value) == msg, (name, str(ei.value), msg)
    # the workspace is still usable after every failure
    A = oracle.gen_matrix(m, k, 1.0, 73)
    B = oracle.gen_matrix(k, n, 1.0, 74)
    assert np.array_equal(oz.os_ii(A, B, 14).C.view(np.uint64), oracle.os_ii(A, B, 14).C.view(np.uint64))
