# round artifacts: GPU tests, smoke, bench line, reference arm, launch list, full captures
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err; echo ref=$?
B="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $B > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r_launches.csv python bench.py $B > /dev/null 2>&1; echo launches=$?
B1="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 -o gpurun_out/r_gemm python bench.py $B1 > /dev/null 2>&1; echo gemm=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"row_scan|col_max|resid_rows|resid_A|crt" -c 6 -o gpurun_out/r_aux python bench.py $B1 > /dev/null 2>&1; echo aux=$?
