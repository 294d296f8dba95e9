# transpose_B write-out rewrite; full captures of resid_A, transpose_B<1>, crt
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:"resid|transpose|crt|row_scan|col_max" -c 12 --csv \
    --log-file gpurun_out/launches_i15.csv python bench.py $B1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"resid_A|transpose_B|crt" -c 4 -o gpurun_out/prof_aux15 python bench.py $B1 > /dev/null 2>&1; echo full=$?
