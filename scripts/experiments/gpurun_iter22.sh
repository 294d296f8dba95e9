# CRT overlapped with the next block's residue GEMM (OZ2G_CRT_OVERLAP)
set -x
mkdir -p gpurun_out
OZ2G_CRT_OVERLAP=4 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_errors_gpu.py -q -x 2>&1 | tail -1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-native"
for r in 1 2; do
  for v in 0 4 8; do
    OZ2G_CRT_OVERLAP=$v timeout 300 python bench.py $B > gpurun_out/ov_${v}_$r.json 2>/dev/null
  done
done
