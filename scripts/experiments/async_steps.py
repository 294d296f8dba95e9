"""Back-to-back asynchronous host-pointer calls at 16384^3: throughput vs the
number of calls in the stream (fill and drain amortised)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02549_b200 as oz
n = 16384
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) - 0.5)
B = (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) - 0.5)
A_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True); A_h.copy_(A)
B_h = torch.empty(B.shape, dtype=torch.float64, pin_memory=True); B_h.copy_(B)
C_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
a, b, c = A_h.numpy(), B_h.numpy(), C_h.numpy()
oz.os_ii(a, b, 16, out=c, blocking=False); oz.synchronize()
for steps in (1, 2, 5, 10):
    t0 = time.perf_counter()
    for _ in range(steps):
        oz.os_ii(a, b, 16, out=c, blocking=False)
    oz.synchronize()
    ms = (time.perf_counter() - t0) / steps * 1e3
    print(f"{steps} calls: {ms:.1f} ms per call ({2 * n**3 / ms / 1e9:.1f} TF/s)", flush=True)
