# multi-device tiling on one GPU, error paths, config sweep
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi_device.py tests/test_errors_gpu.py tests/test_parity_gpu.py -q -rf > gpurun_out/t20.log 2>&1; echo tests=$?
tail -15 gpurun_out/t20.log
timeout 1500 python scripts/configs.py --out gpurun_out/configs_i20.jsonl > gpurun_out/configs_i20.log 2>&1; echo cfg=$?
