mkdir -p gpurun_out
for i in 1 2; do
for ew in 8 4; do
  OZ2G_EPI_WARPS=$ew timeout 300 python scripts/gemm_ab.py | sed "s/^/ew$ew /"
done; done
for ew in 8 4; do
  OZ2G_EPI_WARPS=$ew timeout 300 python scripts/gemm_ab.py --m 2048 --k 65536 | sed "s/^/ew$ew /"
  OZ2G_EPI_WARPS=$ew timeout 300 python scripts/gemm_ab.py --m 4096 | sed "s/^/ew$ew /"
  OZ2G_EPI_WARPS=$ew timeout 300 python scripts/small_overhead2.py 1024 14 | sed "s/^/ew$ew /"
done
