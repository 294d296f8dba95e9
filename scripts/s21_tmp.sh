mkdir -p gpurun_out
cat > /tmp/small.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_02549_b200 as oz
from bench import gen_device
m = int(sys.argv[1]); N = int(sys.argv[2])
A = gen_device(m, m, 0.0, 11, torch.float64, torch.device("cuda", 0))
B = gen_device(m, m, 0.0, 12, torch.float64, torch.device("cuda", 0))
C = torch.empty((m, m), dtype=torch.float64, device="cuda")
for _ in range(6):
    oz.os_ii(A, B, N, out=C)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:"gemm_i8_tc_kernel|resid" -s 12 -c 3 -o gpurun_out/prof_small python /tmp/small.py 1024 14 > /dev/null 2>&1; echo p=$?
