mkdir -p gpurun_out
rm -f /tmp/gemm_ab_ref_*
for cfg in "" "OZ2G_GEMM_FENCE=1" "OZ2G_GEMM=pair" "OZ2G_GEMM=pair OZ2G_GEMM_FENCE=1" "OZ2G_GEMM=pair OZ2G_PAIR_STAGES=6" "OZ2G_GEMM=pair OZ2G_PAIR_STAGES=6 OZ2G_GEMM_FENCE=1" "" "OZ2G_GEMM=pair OZ2G_PAIR_STAGES=6 OZ2G_GEMM_FENCE=1"; do
  env $cfg timeout 300 python scripts/gemm_ab.py
done > gpurun_out/s18_ab.jsonl 2>&1
cat gpurun_out/s18_ab.jsonl
for cfg in "" "OZ2G_GEMM=pair OZ2G_PAIR_STAGES=6 OZ2G_GEMM_FENCE=1"; do
  env $cfg timeout 300 python scripts/gemm_ab.py --m 2048 --k 65536
done >> gpurun_out/s18_ab.jsonl 2>&1
tail -2 gpurun_out/s18_ab.jsonl
