"""e2e (host buffers, blocking calls) per speculation mode on inputs whose
maxima move (phi sweep at 8192^3), plus 16384^3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02549_b200 as oz
from bench import gen_device
dev = torch.device("cuda", 0)
for (m, phi, nmod) in [(8192, 0.0, 12), (8192, 0.5, 12), (8192, 2.0, 12), (8192, 2.0, 16), (8192, 8.0, 12), (16384, 0.0, 16)]:
    A = gen_device(m, m, phi, 11, torch.float64, dev)
    B = gen_device(m, m, phi, 12, torch.float64, dev)
    Ah = torch.empty(A.shape, dtype=torch.float64, pin_memory=True); Ah.copy_(A)
    Bh = torch.empty(B.shape, dtype=torch.float64, pin_memory=True); Bh.copy_(B)
    Ch = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
    a, b, c = Ah.numpy(), Bh.numpy(), Ch.numpy()
    out = []
    for mode in ("2", "1", "0"):
        oz.set_option("spec", int(mode))
        r = oz.os_ii(a, b, nmod, out=c)
        t0 = time.perf_counter()
        for _ in range(3):
            r = oz.os_ii(a, b, nmod, out=c)
        ms = (time.perf_counter() - t0) / 3 * 1e3
        out.append(f"mode {mode}: {ms:6.1f} ms ({2*m**3/ms/1e9:5.1f} TF/s, spec {r.speculation})")
    oz.set_option("spec", -1)
    print(f"{m}^3 phi={phi} N={nmod}: " + " | ".join(out), flush=True)
