set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_blocked_gpu.py tests/test_bounds_gpu.py tests/test_parity_gpu.py -q -rf --tb=short > gpurun_out/t39.log 2>&1; echo t=$?
tail -15 gpurun_out/t39.log
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo bench=$?
