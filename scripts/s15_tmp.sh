python - <<PY
s=open("scripts/prof_fused_dram.sh").read()
i=s.index("cat > /tmp/one_call.py"); j=s.index("PY\n", i)+3
open("/tmp/mk.sh","w").write(s[i:j])
PY
bash /tmp/mk.sh
OZ2G_FUSED=2 timeout 900 ncu --set full --clock-control none -k regex:gemm_crt_fused -s 1 -c 1 -o gpurun_out/prof_fused16k_probe python /tmp/one_call.py 16384 16 > /dev/null 2>&1; echo p=$?
timeout 900 ncu --set full --clock-control none -k regex:"gemm_i8_tc_kernel<1>" -s 2 -c 1 -o gpurun_out/prof_resid16k python /tmp/one_call.py 16384 16 > /dev/null 2>&1; echo r=$?
