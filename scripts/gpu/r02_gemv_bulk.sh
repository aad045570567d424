# bulk-copy dense GEMV (gemv_bulk_kernel): parity tests, isolated prologue timing, same-box decode A/B (HAP_GEMV_BULK=0/1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/bulk_tests.txt 2>&1
tail -3 gpurun_out/bulk_tests.txt
for b in 0 1; do HAP_GEMV_BULK=$b python scripts/diag/fused_norm_bench.py 2>&1 | tail -4 | sed "s/^/bulk=$b /"; done | tee gpurun_out/bulk_iso.txt
for rep in 1 2; do for b in 0 1; do
  HAP_GEMV_BULK=$b python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 2>&1 | tail -1 | sed "s/^/bulk=$b /"
  HAP_GEMV_BULK=$b python scripts/decode_ab.py mixtral-8x7b 1 2 64 2>&1 | tail -1 | sed "s/^/bulk=$b /"
done; done | tee gpurun_out/bulk_ab.txt
