set -x
mkdir -p gpurun_out
OZ2G_GEMM=mcast timeout 600 python -m pytest tests/test_fullsize_gpu.py tests/test_edges_gpu.py tests/test_multi_device.py -q -x 2>&1 | tail -2
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum"
for g in 16 32; do
OZ2G_GEMM=mcast OZ2G_GROUP_M=$g timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv --log-file gpurun_out/mc_$g.csv python bench.py $B1 > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 --csv --log-file gpurun_out/mc_single.csv python bench.py $B1 > /dev/null 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
for r in 1 2 3; do
  timeout 300 python bench.py $B > gpurun_out/ab33_single_$r.json 2>/dev/null
  OZ2G_GEMM=mcast timeout 300 python bench.py $B > gpurun_out/ab33_mc_$r.json 2>/dev/null
done
