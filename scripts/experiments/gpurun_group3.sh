set -x
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2; do for g in 8 16 32; do OZ2G_GROUP_M=$g timeout 300 python bench.py $B > gpurun_out/g3_${g}_$r.json 2>/dev/null; done; done
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for g in 8 16 32; do OZ2G_GROUP_M=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_i8_tc -s 1 -c 2 --csv --log-file gpurun_out/g3_$g.csv python bench.py $B1 > /dev/null 2>&1; done
