# pair GEMM pipeline depth vs DRAM traffic
set -x
mkdir -p gpurun_out
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
OZ2G_GEMM=pair OZ2G_PAIR_STAGES=4 timeout 300 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
for st in 4 6 7; do
OZ2G_GEMM=pair OZ2G_PAIR_STAGES=$st timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/launches_pairS$st.csv python bench.py $B1 > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -c 2 --csv \
    --log-file gpurun_out/launches_single13.csv python bench.py $B1 > /dev/null 2>&1
