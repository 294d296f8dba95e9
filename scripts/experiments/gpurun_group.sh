set -x
mkdir -p gpurun_out
BARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-native"
timeout 300 python bench.py $BARGS > /dev/null 2>&1
for g in 8 16 24 32; do
OZ2G_GROUP_M=$g timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"gemm_i8_tc_kernel<1>" -c 1 --csv \
    --log-file gpurun_out/grp_$g.csv python bench.py $BARGS > /dev/null 2>&1
echo ncu_$g=$?
done
for g in 16 32; do for rep in 1 2; do
  OZ2G_GROUP_M=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/grpb_${g}_$rep.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/grpb_${g}_$rep.json')); print('GRP $g $rep', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
done; done
