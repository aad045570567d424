timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "permute or decode or tiny or qwen" 2>&1 | tail -2
for i in 1 2; do
for v in 0 1; do
HAP_PERMUTE_SMALL=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 | sed "s/^/small=$v /"
HAP_PERMUTE_SMALL=$v timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 64 | sed "s/^/small=$v /"
done
done
