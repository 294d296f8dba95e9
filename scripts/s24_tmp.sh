mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_baseline_configs_gpu.py tests/test_gemm_variants_gpu.py tests/test_graph_gpu.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python scripts/small_overhead2.py 1024 14
timeout 300 python scripts/gemm_ab.py
timeout 300 python scripts/gemm_ab.py --m 4096
timeout 300 python scripts/gemm_ab.py --m 2048 --k 65536
timeout 300 python scripts/timeline.py --m 1024 --moduli 14 --calls 5 --out gpurun_out/tl_1024_s24.json
