timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for g in 0 1; do
HAP_GEMV=$g timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 4 8 64
HAP_GEMV=$g timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 2 4 64
done
done
