# fused decode norm + QKV (hap_rmsnorm_gemm_qkv_rope): parity tests, then a same-box A/B of the
# graph-replayed decode step (HAP_FUSED_NORM=0 vs 1, alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_block_gpu.py tests/test_paged_kv_gpu.py tests/test_kernels_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/fused_tests.txt 2>&1
tail -3 gpurun_out/fused_tests.txt
timeout 600 python -m pytest tests/test_block_gpu.py -m gpu -q -x -k "full_size_mixtral_decode or qwen2_57b_decode_sweep" > gpurun_out/fused_fullsize.txt 2>&1
tail -3 gpurun_out/fused_fullsize.txt
for rep in 1 2; do
  for f in 0 1; do
    HAP_FUSED_NORM=$f python scripts/decode_ab.py qwen2-57b-a14b 1 2 64 2>&1 | sed "s/^/fused=$f /" | tail -1
    HAP_FUSED_NORM=$f python scripts/decode_ab.py mixtral-8x7b 1 2 64 2>&1 | sed "s/^/fused=$f /" | tail -1
  done
done | tee gpurun_out/fused_norm_ab.txt
