set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_errors_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -2
for c in cfg1 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:row_scan --csv \
    --log-file gpurun_out/small4_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"row_scan" -c 2 --csv \
    --log-file gpurun_out/launches_i28.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native > /dev/null 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-native > gpurun_out/bench_i28.json 2>/dev/null
