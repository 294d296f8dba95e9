set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py -q -x 2>&1 | tail -2
for c in cfg1 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/small3_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"resid|transpose|row_scan|col_max|crt" -c 12 --csv \
    --log-file gpurun_out/launches_i27.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native > /dev/null 2>&1
