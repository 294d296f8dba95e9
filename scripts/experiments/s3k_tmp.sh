mkdir -p gpurun_out
R=gpurun_out/s3k
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_errors_gpu.py tests/test_baseline_configs_gpu.py tests/test_bounds_gpu.py -m gpu -q -rf -x > ${R}_tests.log 2>&1; echo tests=$?; tail -3 ${R}_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"crt" -c 2 -o ${R}_crt python bench.py --steps 1 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak > /dev/null 2>&1; echo ncu=$?
timeout 300 python scripts/timeline.py --m 16384 --out ${R}_tl_16k.json > /dev/null 2>&1
