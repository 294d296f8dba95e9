set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_fullsize_gpu.py tests/test_multi_device.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"resid|transpose" -c 6 --csv \
    --log-file gpurun_out/launches_i31.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native > /dev/null 2>&1
for c in cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"resid|transpose" --csv \
    --log-file gpurun_out/small6_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
