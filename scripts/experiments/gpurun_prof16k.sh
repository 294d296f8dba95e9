# launch list of the bench command and a full ncu capture of the residue GEMM at 16384^3, N=16
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
BARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 python bench.py $BARGS > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches16k.csv python bench.py $BARGS > gpurun_out/ncu_launch.log 2>&1
echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_i8_tc_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_gemm16k python bench.py $BARGS > gpurun_out/ncu_full16k.log 2>&1
echo ncu_full=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"resid_A|transpose_B_kernel|crt_kernel|row_scan" -c 5 \
    -o gpurun_out/prof_aux16k python bench.py $BARGS > gpurun_out/ncu_aux16k.log 2>&1
echo ncu_aux=$?
