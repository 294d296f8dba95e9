set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for t in 256 512 1024; do
OZ2G_ROWSCAN_THREADS=$t timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:row_scan -c 2 --csv --log-file gpurun_out/rs_$t.csv python bench.py $B1 > /dev/null 2>&1
done
