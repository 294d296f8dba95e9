# ncu captures of the fused residue-GEMM + CRT kernel and of the two-pass residue GEMM at 4096^3, N = 16
set -x
mkdir -p gpurun_out
cat > /tmp/one_call.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_02549_b200 as oz
from bench import gen_device
m = int(sys.argv[1]); N = int(sys.argv[2])
A = gen_device(m, m, 0.0, 1234, torch.float64, torch.device("cuda", 0))
B = gen_device(m, m, 0.0, 5678, torch.float64, torch.device("cuda", 0))
for _ in range(2):
    oz.os_ii(A, B, N)
torch.cuda.synchronize()
PY
OZ2G_FUSED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_crt_fused -s 1 -c 1 -o gpurun_out/prof_fused python /tmp/one_call.py 4096 16 > gpurun_out/prof_fused.log 2>&1; echo fused=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc_kernel -s 2 -c 1 -o gpurun_out/prof_resid python /tmp/one_call.py 4096 16 > gpurun_out/prof_resid.log 2>&1; echo resid=$?
