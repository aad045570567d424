timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py tests/test_gemv_gpu.py -m gpu -q -x -k "gemm or rope or qwen or decode or tiny or gemv" 2>&1 | tail -2
for i in 1 2; do
for v in 0 1; do HAP_GEMM_SPLIT_DENSE=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 128 256 512 | sed "s/^/sd=$v /"; HAP_GEMM_SPLIT_DENSE=$v timeout 300 python scripts/decode_ab.py mixtral-8x7b 256 512 | sed "s/^/sd=$v /"; done
done
