for m in 2 4; do for v in 0 2; do GEMV_ROWS=$m HAP_GEMV=$v timeout 120 python scripts/gemv_bench.py; done; done
for v in 0 1 0 1; do HAP_GEMV=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 4 8; done
for v in 0 1; do HAP_GEMV=$v timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 8 64; done
