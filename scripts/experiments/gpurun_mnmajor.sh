# MN-major B operand: parity under short timeouts (all three GEMM variants)
set -x
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/mn_single.log 2>&1; echo single=$?
tail -3 gpurun_out/mn_single.log
OZ2G_GEMM=mcast timeout 240 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/mn_mcast.log 2>&1; echo mcast=$?
tail -3 gpurun_out/mn_mcast.log
OZ2G_GEMM=pair timeout 240 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/mn_pair.log 2>&1; echo pair=$?
tail -3 gpurun_out/mn_pair.log
