for p in 0 1 2 3 4 0 2; do HAP_ATTN_POLY=$p timeout 60 python scripts/attn_bench.py; done
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attn_prefill" 2>&1 | tail -2
