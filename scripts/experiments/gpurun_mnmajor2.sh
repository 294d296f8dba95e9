set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/mn_all.log 2>&1; echo tests=$?
tail -3 gpurun_out/mn_all.log
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/mn_launches.csv python bench.py $B1 > /dev/null 2>&1
for r in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-native > gpurun_out/mn_bench_$r.json 2>/dev/null; done
for c in cfg1 cfg2; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mn_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1; done
