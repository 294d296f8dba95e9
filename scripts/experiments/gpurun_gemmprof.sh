# full ncu capture of the residue GEMM and the clearance GEMM (8192^3, N=16)
set -x
mkdir -p gpurun_out
SARGS="--m 8192 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $SARGS > gpurun_out/small.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_i8_tc" -s 2 -c 2 \
    -o gpurun_out/prof_gemm python bench.py $SARGS > gpurun_out/ncu_gemm.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_gemm.log
