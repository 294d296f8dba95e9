# residue-kernel grid sweep (OZ2G_RESID_WAVES) after the sign-interleaved table
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/gpu_tests_i8.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_i8.log
BARGS1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $BARGS1 > /dev/null 2>&1 || exit 1
for v in 0 1 4; do
  OZ2G_RESID_WAVES=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"resid|transpose" -c 6 --csv \
    --log-file gpurun_out/launches_res_$v.csv python bench.py $BARGS1 > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"resid_A|transpose_B_kernel<double, 1>" -c 2 -o gpurun_out/prof_resid2 python bench.py $BARGS1 > gpurun_out/ncu_resid2.log 2>&1
echo ncufull=$?
