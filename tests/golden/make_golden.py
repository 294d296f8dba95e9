"""Regenerates the committed golden fixtures in tests/golden/.

* ref_gen_gemm.npz — outputs of the REFERENCE's own generator (gen.hpp /
  prng.hpp) and INT8 engine (int8gemm.hpp), compiled in place from
  /root/reference by oracle/Makefile into oracle/_ref/liboz2_ref.so.  The
  GPU box has no /root/reference; these fixtures carry the reference's
  behaviour there.
* shift_thresholds.json — the step tables of the scaling exponent derived in
  SURVEY.md §8c (glibc log2), used as golden vectors for both the oracle and
  the product's host-built table.

Run from the repo root:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

GEN_CASES = [  # (rows, cols, phi, seed, dtype)
    (7, 20, 0.0, 0x88, "f64"), (20, 6, 4.0, 0x99, "f64"), (3, 8, 0.5, 0xcc, "f32"),
    (13, 17, 8.0, 0x77, "f64"), (64, 64, 2.0, 12345, "f32"), (1, 1000, 0.0, 1, "f64"),
]


def main():
    R = O.ref_lib()
    if R is None:
        raise SystemExit("oracle/_ref not built: run `make -C oracle` with /root/reference present")
    out = {}
    for idx, (r, c, phi, seed, dt) in enumerate(GEN_CASES):
        arr = np.empty((r, c), dtype=np.float64 if dt == "f64" else np.float32)
        fn = R.ref_gen_matrix_f64 if dt == "f64" else R.ref_gen_matrix_f32
        assert fn(r, c, phi, seed, arr.ctypes.data) == 0
        out[f"gen{idx}"] = arr
    rng = np.random.default_rng(20260214)
    for idx, (m, k, n) in enumerate([(5, 7, 3), (19, 300, 23), (8, 1024, 8)]):
        a = rng.integers(-128, 128, (m, k), dtype=np.int8)
        b = rng.integers(-128, 128, (k, n), dtype=np.int8)
        c = np.empty((m, n), dtype=np.int32)
        assert R.ref_gemm_i8_wrap(m, k, n, a.ctypes.data, b.ctypes.data, c.ctypes.data) == 0
        out[f"gemm{idx}_a"], out[f"gemm{idx}_b"], out[f"gemm{idx}_c"] = a, b, c
    np.savez_compressed(os.path.join(HERE, "ref_gen_gemm.npz"), **out)
    with open(os.path.join(HERE, "gen_cases.json"), "w") as f:
        json.dump(GEN_CASES, f)
    print("wrote", os.path.join(HERE, "ref_gen_gemm.npz"))


if __name__ == "__main__":
    main()
