HAP_GEMM_DEBUG=1 HAP_GEMM_MC=1 timeout 120 python scripts/gemm_l2_sweep.py 2 2>&1 | sort | uniq -c | head -3
HAP_GEMM_MC=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "gemm" 2>&1 | tail -2
for v in 0 1 0 1; do HAP_GEMM_MC=$v timeout 120 python scripts/gemm_l2_sweep.py 10 | sed "s/^/mc=$v /"; done
for v in 0 1 0 1; do HAP_GEMM_MC=$v timeout 120 python scripts/diag/gemm_power.py 4 | sed "s/^/mc=$v /"; done
