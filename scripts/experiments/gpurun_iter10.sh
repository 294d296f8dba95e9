# pair (cta_group::2) vs single-CTA residue GEMM: timed A/B + one full ncu capture each
set -x
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  timeout 300 python bench.py $B > gpurun_out/ab10_single_$r.json 2>/dev/null
  OZ2G_GEMM=pair timeout 300 python bench.py $B > gpurun_out/ab10_pair_$r.json 2>/dev/null
done
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 900 ncu --set full --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 -o gpurun_out/prof_gemm_single python bench.py $B1 > /dev/null 2>&1; echo s=$?
OZ2G_GEMM=pair timeout 900 ncu --set full --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 -o gpurun_out/prof_gemm_pair python bench.py $B1 > /dev/null 2>&1; echo p=$?
nvidia-smi -q -d POWER > gpurun_out/power_q.txt 2>&1
