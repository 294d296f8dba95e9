# long-row scan (one row per SM, 4 first-pass steps in flight): parity, cfg5 launch list, 16384^3 bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_edges_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -3
BARGS="--m 2048 --k 65536 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 python bench.py $BARGS > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_cfg5_rowscan2.csv python bench.py $BARGS > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_cfg5.json')); print(d['value'], d['ms_per_step'], d['stages_ms'])"
python scripts/launches.py gpurun_out/launches_cfg5_rowscan2.csv | grep -v "at::"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/bench_16k.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_16k.json')); print(d['value'], d['ms_per_step'], d['stages_ms'])"
