# early A residues in the pipelined host path, split tail; error-path tests; config sweep; bench e2e
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_errors_gpu.py tests/test_parity_gpu.py tests/test_cpp_dropin.py -q -rf > gpurun_out/t19.log 2>&1; echo tests=$?
tail -5 gpurun_out/t19.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-native > gpurun_out/bench_i19.json 2>gpurun_out/bench_i19.err; echo bench=$?
timeout 1500 python scripts/configs.py --out gpurun_out/configs_i19.jsonl > gpurun_out/configs_i19.log 2>&1; echo cfg=$?
