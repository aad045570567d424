timeout 900 python -m pytest tests/test_block_gpu.py tests/test_kernels_gpu.py -m gpu -q -x -k "qwen or shared or gemm or decode" 2>&1 | tail -2
for i in 1 2 3; do
HAP_SHARED_SMS=0 timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 512 | sed "s/^/sh=all /"
timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 512 | sed "s/^/sh=half /"
done
HAP_SHARED_SMS=0 timeout 300 python scripts/decode_ab.py qwen1.5-moe-a2.7b 1 8 64 | sed "s/^/sh=all /"
timeout 300 python scripts/decode_ab.py qwen1.5-moe-a2.7b 1 8 64 | sed "s/^/sh=half /"
