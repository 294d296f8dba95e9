# transpose_B grid order; full capture of the B residue transpose
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:"resid|transpose|crt|row_scan|col_max" -c 12 --csv \
    --log-file gpurun_out/launches_i14.csv python bench.py $B1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:transpose_B -s 1 -c 1 -o gpurun_out/prof_tB1 python bench.py $B1 > /dev/null 2>&1; echo full=$?
