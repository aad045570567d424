for i in 1 2 3; do
for g in 0 1; do
HAP_GEMV=$g timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8
HAP_GEMV=$g timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 2 8
done
done
