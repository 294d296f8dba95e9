set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2 3; do
  timeout 300 python bench.py $B > gpurun_out/wb_block_$r.json 2>/dev/null
  OZ2G_WBLOCK_MIN_MB=100000 timeout 300 python bench.py $B > gpurun_out/wb_full_$r.json 2>/dev/null
done
for c in cfg1 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crt --csv --log-file gpurun_out/crt37_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
