"""Blocking host-pointer calls at 16384^3: speculated row + column exponents (2), column only (1), none (0)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2602_02549_b200 as oz
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) - 0.5)
B = (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) - 0.5)
A_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True); A_h.copy_(A)
B_h = torch.empty(B.shape, dtype=torch.float64, pin_memory=True); B_h.copy_(B)
C_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
a, b, c = A_h.numpy(), B_h.numpy(), C_h.numpy()
for spec in ["2", "1", "0", "2", "1", "0", "2"]:
    oz.set_option("spec", int(spec))
    t0 = time.perf_counter()
    r = oz.os_ii(a, b, 16, out=c)
    print(f"spec={spec} speculation={r.speculation} {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
names = ["h2d", "scale", "clearance", "expo", "resid", "gemm", "crt", "d2h"]
for spec in ["2", "1"]:
    oz.set_option("spec", int(spec))
    r = oz.os_ii(a, b, 16, out=c, timing=True)
    print(f"spec={spec} busy ms:", {nm: round(v, 2) for nm, v in zip(names, r.stage_ms)}, "launches", r.kernels_launched)
