set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "gemm or rope" 2>&1 | tail -3
for m in 1 8; do for v in 0 2 0 2; do GEMV_ROWS=$m HAP_GEMV=$v timeout 120 python scripts/gemv_bench.py; done; done
