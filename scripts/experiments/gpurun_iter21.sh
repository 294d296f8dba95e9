# L2 eviction hints one operand at a time, raster group 16 / 32: residue-GEMM DRAM bytes + timed runs
set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
timeout 300 python bench.py $B1 > /dev/null 2>&1 || exit 1
for cfg in "0 16" "2 16" "3 16" "2 32" "0 32"; do
  set -- $cfg
  OZ2G_L2HINT=$1 OZ2G_GROUP_M=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/l2h_$1_$2.csv python bench.py $B1 > /dev/null 2>&1
done
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  for cfg in "0 16" "2 16" "2 32"; do
    set -- $cfg
    OZ2G_L2HINT=$1 OZ2G_GROUP_M=$2 timeout 300 python bench.py $B > gpurun_out/l2hb_$1_$2_$r.json 2>/dev/null
  done
done
