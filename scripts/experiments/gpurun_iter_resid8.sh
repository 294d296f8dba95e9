# residue writers unrolled over 8 moduli: parity + launch list at 16384^2 and 2048x65536
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_fuzz_gpu.py -x -q 2>&1 | tail -3
BARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 python bench.py $BARGS > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_resid8.csv python bench.py $BARGS > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
cat gpurun_out/bench_iter.json
python scripts/launches.py gpurun_out/launches_resid8.csv
