# two-pass row scan CTA size at 16384^2 (OZ2G_ROWSCAN_THREADS 256 / 512 / 1024): parity + launch lists
set -x
mkdir -p gpurun_out
for t in 512 256; do OZ2G_ROWSCAN_THREADS=$t timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1; done
BARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for t in 1024 512 256; do
  OZ2G_ROWSCAN_THREADS=$t timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:row_scan -c 5 --csv \
    --log-file gpurun_out/launches_rowscan_t$t.csv python bench.py $BARGS > /dev/null 2>&1
  echo t=$t; python scripts/launches.py gpurun_out/launches_rowscan_t$t.csv | tail -1
done
