set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_bounds_gpu.py -q -x 2>&1 | tail -2
for c in cfg1 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"crt|row_scan" --csv \
    --log-file gpurun_out/small5_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"crt|row_scan" -c 4 --csv \
    --log-file gpurun_out/launches_i29.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native > /dev/null 2>&1
