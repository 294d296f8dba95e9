set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/t30.log 2>&1; echo tests=$?
tail -3 gpurun_out/t30.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-native > gpurun_out/bench_i30.json 2>gpurun_out/bench_i30.err; echo b=$?
timeout 300 python scripts/configs.py --out gpurun_out/configs_i30.jsonl > /dev/null 2>&1; echo c=$?
