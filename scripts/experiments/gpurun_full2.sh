set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -rA 2>&1 | grep -E "PASS|FAIL|passed|failed|Error" | tail -40
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
