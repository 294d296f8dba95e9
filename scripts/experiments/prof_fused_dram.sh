# DRAM bytes and duration of the fused kernel vs the two-pass residue GEMM at 16384^3, N = 16
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
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second"
OZ2G_FUSED=2 timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_crt_fused -s 1 -c 1 --csv python /tmp/one_call.py 16384 16 > gpurun_out/prof_fused_dram.csv 2> gpurun_out/prof_fused_dram.err; echo fused=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 10 -c 1 --csv python /tmp/one_call.py 16384 16 > gpurun_out/prof_resid_dram.csv 2> gpurun_out/prof_resid_dram.err; echo resid=$?
