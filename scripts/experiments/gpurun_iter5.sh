set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for g in 8 16 32; do
  OZ2G_GROUP_M=$g timeout 300 python bench.py --m 8192 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/g$g.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/g$g.json')); print('group', $g, d['ms_per_step'], d['stages_ms']['residue_gemms'])"
done
SARGS="--m 8192 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for g in 8 32; do
OZ2G_GROUP_M=$g timeout 300 python bench.py $SARGS > gpurun_out/small_$g.json 2>&1 && \
OZ2G_GROUP_M=$g timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_i8_tc" -c 4 --csv \
    --log-file gpurun_out/gemm_dram_$g.csv python bench.py $SARGS > /dev/null 2>&1
echo ncu_$g=$?
done
