set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_bounds_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:crt -c 16 --csv --log-file gpurun_out/crt36.csv python bench.py $B1 > /dev/null 2>&1
for c in cfg1 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crt --csv --log-file gpurun_out/crt36_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
