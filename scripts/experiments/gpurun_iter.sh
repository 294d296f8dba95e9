# one build->measure iteration on the B200: parity, bench, ncu launch list
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -5
BARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 python bench.py $BARGS > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py $BARGS > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
cat gpurun_out/bench_iter.json
