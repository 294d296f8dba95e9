set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_bounds_gpu.py -x -q 2>&1 | tail -3
for rep in 1 2; do
for h in 1 0; do
  OZ2G_L2HINT=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/hint_${h}_$rep.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/hint_${h}_$rep.json')); print('HINT $h $rep', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['stages_ms']['residue_gemms'])"
done
done
BARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $BARGS > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_i8_tc" -c 4 --csv \
    --log-file gpurun_out/gemm_dram_hint.csv python bench.py $BARGS > /dev/null 2>&1
echo ncu=$?
