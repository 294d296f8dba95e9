set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
BARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $BARGS > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_i6.csv python bench.py $BARGS > /dev/null 2>&1
echo ncu=$?
timeout 900 python bench.py > gpurun_out/bench_i6.json 2> gpurun_out/bench_i6.err; echo rc=$?
cat gpurun_out/bench_i6.json
