mkdir -p gpurun_out
R=gpurun_out/r2
B1="--steps 1 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc -s 1 -c 1 -o ${R}_gemm python bench.py $B1 > /dev/null 2>&1; echo gemm=$?
B="--steps 2 --warmup 3 --moduli 16 --no-cpu-baseline --no-e2e --no-native --no-int8-peak"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file ${R}_launches_b.csv python bench.py $B > /dev/null 2>&1; echo launches=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file ${R}_launches_cfg5.csv python bench.py $B --m 2048 --k 65536 > /dev/null 2>&1; echo launches5=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"resid_A|resid_rows" -s 3 -c 2 -o ${R}_resid_cfg5 python bench.py $B1 --m 2048 --k 65536 > /dev/null 2>&1; echo resid5=$?
timeout 900 python scripts/configs.py --out ${R}_configs.jsonl > /dev/null 2>&1; echo configs=$?
