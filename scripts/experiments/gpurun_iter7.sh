# parity suite, launch list with DRAM bytes, CRT conversion-split sweep, full bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short > gpurun_out/gpu_tests_i7.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests_i7.log
BARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for v in 0 3 5 8; do
  OZ2G_CRT_NFP=$v timeout 300 python bench.py $BARGS > gpurun_out/crt_nfp_$v.json 2>/dev/null
done
BARGS1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_i7.csv python bench.py $BARGS1 > /dev/null 2>&1
echo ncu=$?
for v in 0 8; do
  OZ2G_CRT_NFP=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:crt_kernel -c 2 --csv \
    --log-file gpurun_out/launches_crt_$v.csv python bench.py $BARGS1 > /dev/null 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_i7.json 2> gpurun_out/bench_i7.err; echo rc=$?
cat gpurun_out/bench_i7.json
