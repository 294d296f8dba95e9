# pair GEMM raster sweep (group_m in pair tiles) vs single at group 16
set -x
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  timeout 300 python bench.py $B > gpurun_out/ab11_single16_$r.json 2>/dev/null
  for g in 4 6 8; do
    OZ2G_GEMM=pair OZ2G_GROUP_M=$g timeout 300 python bench.py $B > gpurun_out/ab11_pair${g}_$r.json 2>/dev/null
  done
done
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for g in 4 8; do
OZ2G_GEMM=pair OZ2G_GROUP_M=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/launches_pair$g.csv python bench.py $B1 > /dev/null 2>&1
done
