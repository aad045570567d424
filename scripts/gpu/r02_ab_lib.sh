# A/B of the working-tree library against ab_lib/old.so (the previous commit's build)
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_gemv_gpu.py -m gpu -q -x -k "gemm or rope or gemv" 2>&1 | tail -2
for i in 1 2 3; do
HAP_KERNELS_LIB=$PWD/ab_lib/old.so timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 64 | sed 's/^/old /'
timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 64 | sed 's/^/new /'
HAP_KERNELS_LIB=$PWD/ab_lib/old.so timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 64 | sed 's/^/old /'
timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 64 | sed 's/^/new /'
done
