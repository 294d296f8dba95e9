# multicast-B GEMM variant: parity under a short timeout first
set -x
mkdir -p gpurun_out
OZ2G_GEMM=mcast timeout 240 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/t32.log 2>&1; echo t=$?
tail -5 gpurun_out/t32.log
