# prefetching residue writers
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:"resid|transpose|crt|row_scan|col_max" -c 12 --csv \
    --log-file gpurun_out/launches_i18.csv python bench.py $B1 > /dev/null 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/bench_i18.json 2>/dev/null
