for e in 0 2 1 0 2; do HAP_ATTN_EMU=$e timeout 60 python scripts/attn_bench.py; done
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attn_prefill" 2>&1 | tail -2
