"""e2e per speculation mode on the smaller BASELINE configs (cfg2 SGEMM 4096^3,
4096^3 DGEMM, cfg5 2048 x 65536 x 2048)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02549_b200 as oz
from bench import gen_device
dev = torch.device("cuda", 0)
for (m, k, n, dt, nmod) in [(4096, 4096, 4096, torch.float32, 6), (4096, 4096, 4096, torch.float64, 14),
                            (2048, 65536, 2048, torch.float64, 16), (8192, 8192, 8192, torch.float64, 16)]:
    A = gen_device(m, k, 0.0, 11, dt, dev)
    B = gen_device(k, n, 0.0, 12, dt, dev)
    Ah = torch.empty(A.shape, dtype=dt, pin_memory=True); Ah.copy_(A)
    Bh = torch.empty(B.shape, dtype=dt, pin_memory=True); Bh.copy_(B)
    Ch = torch.empty((m, n), dtype=dt, pin_memory=True)
    a, b, c = Ah.numpy(), Bh.numpy(), Ch.numpy()
    out = []
    for mode in ("2", "1", "0"):
        oz.set_option("spec", int(mode))
        r = oz.os_ii(a, b, nmod, out=c); r = oz.os_ii(a, b, nmod, out=c)
        t0 = time.perf_counter()
        for _ in range(5):
            r = oz.os_ii(a, b, nmod, out=c)
        ms = (time.perf_counter() - t0) / 5 * 1e3
        out.append(f"mode {mode}: {ms:6.2f} ms ({2*m*n*k/ms/1e9:5.1f} TF/s, spec {r.speculation})")
    oz.set_option("spec", -1)
    print(f"{m}x{k}x{n} {str(dt)[6:]} N={nmod}: " + " | ".join(out), flush=True)
