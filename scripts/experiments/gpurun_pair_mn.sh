set -x
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  timeout 300 python bench.py $B > gpurun_out/pmn_single_$r.json 2>/dev/null
  OZ2G_GEMM=pair OZ2G_PAIR_STAGES=4 OZ2G_GROUP_M=8 timeout 300 python bench.py $B > gpurun_out/pmn_p4_$r.json 2>/dev/null
  OZ2G_GEMM=pair OZ2G_PAIR_STAGES=5 OZ2G_GROUP_M=8 timeout 300 python bench.py $B > gpurun_out/pmn_p5_$r.json 2>/dev/null
  OZ2G_GEMM=mcast timeout 300 python bench.py $B > gpurun_out/pmn_mc_$r.json 2>/dev/null
done
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for v in "pair 4" "pair 5" "mcast 4"; do set -- $v
OZ2G_GEMM=$1 OZ2G_PAIR_STAGES=$2 OZ2G_GROUP_M=8 timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv --log-file gpurun_out/pmn_$1$2.csv python bench.py $B1 > /dev/null 2>&1
done
