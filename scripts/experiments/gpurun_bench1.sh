set -x
mkdir -p gpurun_out
timeout 300 python bench.py --m 4096 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
