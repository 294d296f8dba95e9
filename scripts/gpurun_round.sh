# Round artifacts on one B200 (gpurun -- 'bash scripts/gpurun_round.sh'): GPU test suite, smoke(),
# the default bench line, the reference arm, the launch list, ncu --set full captures of the residue GEMM,
# the auxiliary kernels at 16384^3 and cfg5, the INT8 peak, every BASELINE config, the multi-GPU tile
# projection and kernel timelines.  Outputs in gpurun_out/r2_*; the summaries go to profiles/.
set -x
mkdir -p gpurun_out
R=gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -rf > ${R}_tests.log 2>&1; echo tests=$?
tail -3 ${R}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${R}_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > ${R}_bench.json 2> ${R}_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${R}_bench_ref.json 2> ${R}_bench_ref.err; echo ref=$?
timeout 300 python scripts/int8_peak.py --out ${R}_int8_peak.json > /dev/null 2>&1; echo peak=$?
B="--steps 2 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file ${R}_launches.csv python bench.py $B > /dev/null 2>&1; echo launches=$?
B1="--steps 1 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 -o ${R}_gemm python bench.py $B1 > /dev/null 2>&1; echo gemm=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"row_scan|col_max|resid_rows|resid_A|crt" -c 6 -o ${R}_aux python bench.py $B1 > /dev/null 2>&1; echo aux=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"row_scan|col_max|resid_rows|resid_A|crt" -c 6 -o ${R}_aux_cfg5 python bench.py $B1 --m 2048 --k 65536 > /dev/null 2>&1; echo aux5=$?
B5="--steps 2 --warmup 3 --moduli 16 --m 2048 --k 65536 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file ${R}_launches_cfg5.csv python bench.py $B5 > /dev/null 2>&1; echo launches5=$?
timeout 900 python scripts/configs.py --out ${R}_configs.jsonl > /dev/null 2>&1; echo configs=$?
timeout 900 python scripts/experiments/tile_projection.py > ${R}_tile_projection.jsonl 2>/dev/null; echo proj=$?
timeout 300 python scripts/timeline.py --m 16384 --out ${R}_tl_16384.json > /dev/null 2>&1; echo tl=$?
timeout 300 python scripts/timeline.py --m 1024 --moduli 14 --calls 5 --out ${R}_tl_1024.json > /dev/null 2>&1; echo tl1=$?
