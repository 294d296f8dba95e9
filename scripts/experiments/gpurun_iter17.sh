set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $B1 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"transpose_B|resid_A" -c 3 -o gpurun_out/prof_tB2 python bench.py $B1 > /dev/null 2>&1; echo full=$?
