set -x
mkdir -p gpurun_out
OZ2G_CRT_CV=4 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_blocked_gpu.py tests/test_bounds_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for cv in 4 8; do
OZ2G_CRT_CV=$cv timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:crt -c 8 --csv --log-file gpurun_out/cv_$cv.csv python bench.py $B1 > /dev/null 2>&1
for c in cfg1 cfg2; do
  OZ2G_CRT_CV=$cv timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crt --csv --log-file gpurun_out/cv_${cv}_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
done
