mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_baseline_configs_gpu.py tests/test_speculation_gpu.py tests/test_fuzz_gpu.py tests/test_edges_gpu.py -m gpu -q -x 2>&1 | tail -2
B="--steps 2 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"resid" -c 40 --csv --log-file gpurun_out/s26_launches.csv python bench.py $B > /dev/null 2>&1; echo l=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"resid" -c 40 --csv --log-file gpurun_out/s26_launches5.csv python bench.py $B --m 2048 --k 65536 > /dev/null 2>&1; echo l5=$?
timeout 300 python scripts/gemm_ab.py
timeout 300 python scripts/gemm_ab.py --m 2048 --k 65536
