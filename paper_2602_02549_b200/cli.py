"""Command-line front end mirroring the reference CLI (tools/oz2emu.cpp:193-285).

    python -m paper_2602_02549_b200.cli table --n 20 --mode fp64 [--out F]
    python -m paper_2602_02549_b200.cli emulate --a A.mat --b B.mat --n 20 --mode fp64 --out C.mat
    python -m paper_2602_02549_b200.cli bounds --a A.mat --b B.mat --n 20 --mode fp64 [--tight]
    python -m paper_2602_02549_b200.cli suggest-n --a A.mat --b B.mat --target 1e-12 --mode fp64
    python -m paper_2602_02549_b200.cli experiment --m 64 --n 64 --k 1024 --phi 0.5 2 8 --mode fp64 --out sweep.csv
    python -m paper_2602_02549_b200.cli selftest

Same options, output formats and exit codes (2 on an exception); the
computation runs on the GPU through the library.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

from . import emulate as E
from .matrix_io import hexfloat, read_matrix, write_matrix


def _mode(s: str) -> int:
    if s == "fp32":
        return E.F32
    if s == "fp64":
        return E.F64
    raise RuntimeError(f"unknown mode '{s}' (expected fp32|fp64)")


def _dump_table(t: E.ModuliTable, out) -> None:  # oz2emu.cpp:37-46
    out.write(f"P={t.P},rho={t.rho},P1={hexfloat(t.P1)},P2={hexfloat(t.P2)},P_inv={hexfloat(t.P_inv)},"
              f"P_prime={hexfloat(float(t.P_prime))}\n")
    out.write("ell,p,q,beta,s1,s2\n")
    for l in range(t.n):
        out.write(f"{l + 1},{t.p[l]},{t.q[l]},{t.beta[l]},{hexfloat(t.s1[l])},{hexfloat(t.s2[l])}\n")


def _load_pair(a_path, b_path, mode):  # oz2emu.cpp:52-59
    a, b = read_matrix(a_path), read_matrix(b_path)
    want = np.float32 if mode == E.F32 else np.float64
    if a.dtype != want or b.dtype != want:
        names = {np.dtype(np.float32): "fp32", np.dtype(np.float64): "fp64"}
        raise RuntimeError(f"mode mismatch: --mode is {'fp32' if mode == E.F32 else 'fp64'} but inputs are "
                           f"{names[a.dtype]}/{names[b.dtype]}")
    return a, b


def cmd_selftest() -> int:
    """Device self-checks drawn from the reference's emulate tests."""
    checks = []
    one = np.ones((1, 1))
    r = E.os_ii(one, one, 2, keep_intermediates=True)
    checks.append(("1x1 hand trace at N=2 (C=1, mu=nu=7, W=(0,64))",
                   r.C[0, 0] == 1.0 and r.scaling.mu[0] == 7 and list(r.crt.W[:, 0, 0]) == [0, 64]))
    checks.append(("|C-1| <= 2^-40 for N=10,30,49",
                   all(abs(E.os_ii(one, one, n).C[0, 0] - 1.0) <= 2.0 ** -40 for n in (10, 30, 49))))
    try:
        E.os_ii(np.full((3, 8), 0.3, np.float32), np.full((8, 3), 0.7, np.float32), E.fp32_safe_moduli_max() + 1)
        ok = False
    except E.RangeError:
        ok = True
    checks.append(("fp32 range error beyond the ceiling", ok))
    a = np.sin(np.arange(9 * 40, dtype=np.float64)).reshape(9, 40)
    b = np.cos(np.arange(40 * 9, dtype=np.float64)).reshape(40, 9)
    checks.append(("repeated calls bit-identical", E.os_ii(a, b, 25).C.tobytes() == E.os_ii(a, b, 25).C.tobytes()))
    z = np.zeros((2, 3))
    z[0] = 1.0
    try:
        E.os_ii(z, np.ones((3, 2)), 5)
        ok = False
    except E.DomainError:
        ok = True
    checks.append(("zero row rejected (domain_error)", ok))
    for name, ok in checks:
        print(f"[{'PASS' if ok else 'FAIL'}] {name}")
    good = all(ok for _, ok in checks)
    print("selftest: all suites passed" if good else "selftest: FAILURES detected")
    return 0 if good else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="oz2g", description="CRT-based FP32/FP64 GEMM emulation on B200 INT8 tensor cores")
    ap.add_argument("--threads", type=int, default=0, help="accepted for compatibility (GPU execution)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("table")
    t.add_argument("--n", type=int, required=True)
    t.add_argument("--mode", required=True)
    t.add_argument("--out", default="")
    e = sub.add_parser("emulate")
    for opt in ("--a", "--b", "--mode", "--out"):
        e.add_argument(opt, required=True)
    e.add_argument("--n", type=int, required=True)
    b = sub.add_parser("bounds")
    for opt in ("--a", "--b", "--mode"):
        b.add_argument(opt, required=True)
    b.add_argument("--n", type=int, required=True)
    b.add_argument("--tight", action="store_true")
    s = sub.add_parser("suggest-n")
    for opt in ("--a", "--b", "--mode"):
        s.add_argument(opt, required=True)
    s.add_argument("--target", type=float, required=True)
    x = sub.add_parser("experiment")
    x.add_argument("--m", type=int, default=64)
    x.add_argument("--n", type=int, default=64)
    x.add_argument("--k", type=int, default=1024)
    x.add_argument("--phi", type=float, nargs="+", default=[0.5, 2.0, 8.0])
    x.add_argument("--mode", required=True)
    x.add_argument("--n-list", type=int, nargs="+", default=None)
    x.add_argument("--seed", type=int, default=1)
    x.add_argument("--trials", type=int, default=1)
    x.add_argument("--out", required=True)
    sub.add_parser("selftest").add_argument("--deep", action="store_true")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "table":
            tab = E.table_for(args.n, _mode(args.mode))
            if args.out:
                with open(args.out, "w") as f:
                    _dump_table(tab, f)
            else:
                _dump_table(tab, sys.stdout)
            return 0
        if args.cmd == "emulate":  # oz2emu.cpp:61-74
            mode = _mode(args.mode)
            a, bm = _load_pair(args.a, args.b, mode)
            res = E.os_ii(a, bm, args.n)
            write_matrix(args.out, res.C)
            if res.subnormal:
                print("note: some outputs passed through the subnormal range", file=sys.stderr)
            return 0
        if args.cmd == "bounds":  # oz2emu.cpp:76-107
            mode = _mode(args.mode)
            a, bm = _load_pair(args.a, args.b, mode)
            res = E.os_ii(a, bm, args.n, bounds="full")
            bnd = res.bounds["tight" if args.tight else "cheap"]
            mx, mn = float(bnd.max()), float(bnd.min())
            print(f"bound={'tight' if args.tight else 'cheap'} n={args.n} max={hexfloat(mx)} ({mx:.17g}) "
                  f"min={hexfloat(mn)} ({mn:.17g})")
            return 0
        if args.cmd == "suggest-n":  # oz2emu.cpp:109-124
            mode = _mode(args.mode)
            a, bm = _load_pair(args.a, args.b, mode)
            r = E.suggest_n(a, bm, args.target)
            if r.achievable:
                print(f"n={r.n} cheap_bound_max={hexfloat(r.bound_max)} ({r.bound_max:.17g})")
                return 0
            cap = E.fp32_safe_moduli_max() if mode == E.F32 else 49
            print(f"not achievable with N <= {cap}; best cheap_bound_max={hexfloat(r.bound_max)} ({r.bound_max:.17g})")
            return 1
        if args.cmd == "experiment":  # oz2emu.cpp:126-144
            from .experiment import ExperimentConfig, run_experiment, write_experiment_csv
            mode = _mode(args.mode)
            n_list = args.n_list
            if not n_list:
                cap = E.fp32_safe_moduli_max() if mode == E.F32 else 49
                n_list = list(range(2, cap + 1))
            violations = 0
            for phi in args.phi:
                cfg = ExperimentConfig(m=args.m, n=args.n, k=args.k, phi=phi, mode=mode, n_list=n_list,
                                       seed=args.seed, trials=args.trials)
                rows = run_experiment(cfg)
                path = args.out
                if len(args.phi) > 1:
                    suffix = f".phi{phi:g}"
                    path = path[:-4] + suffix + ".csv" if path.endswith(".csv") else path + suffix
                write_experiment_csv(path, rows)
                for r in rows:
                    if not (r.err_max <= r.est_max <= r.est2_max and r.err_min <= r.est_min):
                        print(f"invariant violation at phi={phi:g} n={r.n}", file=sys.stderr)
                        violations += 1
                print(f"wrote {path} ({len(rows)} rows)")
            return 0 if violations == 0 else 1
        if args.cmd == "selftest":
            return cmd_selftest()
    except Exception as ex:  # oz2emu.cpp:280-283
        print(f"error: {ex}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
