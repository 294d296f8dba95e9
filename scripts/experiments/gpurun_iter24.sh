# EVICT_LAST on A with an L2 persisting carve-out
set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
OZ2G_L2PERSIST_MB=32 timeout 300 python bench.py $B1 2>&1 | grep -i persist
for cfg in "2 32 16" "2 48 16" "2 64 16" "2 64 32" "0 64 16"; do
  set -- $cfg
  OZ2G_L2HINT=$1 OZ2G_L2PERSIST_MB=$2 OZ2G_GROUP_M=$3 timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv \
    --log-file gpurun_out/lp_$1_$2_$3.csv python bench.py $B1 > /dev/null 2>&1
done
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  timeout 300 python bench.py $B > gpurun_out/lpb_base_$r.json 2>/dev/null
  OZ2G_L2HINT=2 OZ2G_L2PERSIST_MB=64 timeout 300 python bench.py $B > gpurun_out/lpb_p64_$r.json 2>/dev/null
done
