for v in 0 2 1 0 2 1; do HAP_GEMM_NOLOAD=$v timeout 120 python scripts/diag/gemm_power.py 4; done 2>&1 | grep noload
