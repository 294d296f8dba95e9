set -x
mkdir -p gpurun_out
OZ2G_GEMM=pair timeout 300 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -8
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in single pair; do
  OZ2G_GEMM=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/v_$v.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/v_$v.json')); print('$v', d['value'], d['ms_per_step'], d['stages_ms'], d['clocks'])"
done
for g in 32 64; do
  OZ2G_GROUP_M=$g OZ2G_GEMM=pair timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/pg$g.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/pg$g.json')); print('pair group $g', d['value'], d['ms_per_step'], d['stages_ms']['residue_gemms'])"
done
