set -x
mkdir -p gpurun_out
for c in cfg1 cfg2; do
  timeout 300 python scripts/small_configs.py $c || exit 1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size --clock-control none --csv \
    --log-file gpurun_out/small_$c.csv python scripts/small_configs.py $c > /dev/null 2>&1
done
