set -x
mkdir -p gpurun_out
timeout 900 python scripts/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain=$?
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck=$?
OZ2G_WBLOCK_MIN_MB=0 timeout 1200 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_memcheck_blocked.log 2>&1; echo memcheck_blocked=$?
OZ2G_GEMM=pair timeout 1200 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_memcheck_pair.log 2>&1; echo memcheck_pair=$?
OZ2G_GEMM=mcast timeout 1200 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_memcheck_mcast.log 2>&1; echo memcheck_mcast=$?
