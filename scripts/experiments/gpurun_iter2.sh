# parity + bench + launch list + full ncu capture of the residue kernels
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -5
BARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 python bench.py $BARGS > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py $BARGS > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
SARGS="--m 8192 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $SARGS > gpurun_out/small.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"resid_A|transpose_B_kernel|crt_kernel|row_scan" -c 5 \
    -o gpurun_out/prof_resid python bench.py $SARGS > gpurun_out/ncu_full.log 2>&1
echo ncu_full_rc=$?
cat gpurun_out/bench_iter.json
