set -x
mkdir -p gpurun_out
nvidia-smi -q -d POWER | grep -iE "limit|draw" | head -12
nvidia-smi -q -d CLOCK | grep -iE "graphics|sm " | head -8
for rep in 1 2 3; do
for v in single pair; do
  OZ2G_GEMM=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/ab_${v}_$rep.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab_${v}_$rep.json')); print('AB $v $rep', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
done
done
