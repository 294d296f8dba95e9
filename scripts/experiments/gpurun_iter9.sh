# E'-bucketed residue tables: parity + residue kernel launch list + stage timing
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/gpu_tests_i9.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_i9.log
BARGS1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/bench_i9.json 2>/dev/null || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:"resid|transpose" -c 6 --csv \
    --log-file gpurun_out/launches_res_i9.csv python bench.py $BARGS1 > /dev/null 2>&1
echo ncu=$?
