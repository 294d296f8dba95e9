# pair GEMM: stages x raster group; DRAM, tensor-active, clock per config
set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 300 python bench.py $B1 > /dev/null 2>&1 || exit 1
for cfg in "4 8" "5 8" "5 16" "6 12" "5 12"; do
  set -- $cfg
  OZ2G_GEMM=pair OZ2G_PAIR_STAGES=$1 OZ2G_GROUP_M=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv \
    --log-file gpurun_out/pp_$1_$2.csv python bench.py $B1 > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv --log-file gpurun_out/pp_single.csv python bench.py $B1 > /dev/null 2>&1
