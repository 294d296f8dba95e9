mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x -m gpu 2>&1 | tail -2
AB_MODES=0,2,1 timeout 400 python scripts/fused_ab.py 16384x16384x16384x16 2048x65536x2048x16 4096x4096x4096x16 > gpurun_out/s13_ab.jsonl 2>&1; echo ab=$?; cut -c1-160 gpurun_out/s13_ab.jsonl
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"
OZ2G_FUSED=1 timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_crt_fused -s 1 -c 1 --csv python /tmp/one_call.py 16384 16 2>/dev/null | tail -3 | cut -c150-400
