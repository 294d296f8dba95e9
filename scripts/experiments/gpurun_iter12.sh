# raster along N (OZ2G_GROUP_N) for pair and single residue GEMMs: DRAM bytes + timed runs
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for g in 4 8 16; do
OZ2G_GEMM=pair OZ2G_GROUP_N=$g timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/launches_pairN$g.csv python bench.py $B1 > /dev/null 2>&1
done
for g in 8 16; do
OZ2G_GROUP_N=$g timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/launches_singleN$g.csv python bench.py $B1 > /dev/null 2>&1
done
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do
  timeout 300 python bench.py $B > gpurun_out/ab12_single_$r.json 2>/dev/null
  OZ2G_GEMM=pair OZ2G_GROUP_N=8 timeout 300 python bench.py $B > gpurun_out/ab12_pairN8_$r.json 2>/dev/null
done
