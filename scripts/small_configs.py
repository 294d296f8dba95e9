"""Back-to-back os_ii calls on the BASELINE configs that fit a quick run (cfg1, cfg2, cfg5; for ncu launch lists)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_02549_b200 as oz  # noqa: E402
from bench import gen_device  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dev = torch.device("cuda", 0)
if which == "cfg1":
    m = n = k = 1024; N = 14; dt = torch.float64
elif which == "cfg5":
    m = n = 2048; k = 65536; N = 16; dt = torch.float64
else:
    m = n = k = 4096; N = 6; dt = torch.float32
A = gen_device(m, k, 0.0, 1, dt, dev)
B = gen_device(k, n, 0.0, 2, dt, dev)
C = torch.empty((m, n), dtype=dt, device=dev)
for _ in range(4):
    oz.os_ii(A, B, N, out=C)
torch.cuda.synchronize()
