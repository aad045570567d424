mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemv_gpu.py -m gpu -q -x 2>&1 | tail -2
for a in 0 1; do HAP_GEMV_ASYNC=$a python scripts/diag/fused_norm_bench.py 2>&1 | tail -4 | sed "s/^/async=$a /"; done
for rep in 1 2; do for a in 0 1; do
  HAP_GEMV_ASYNC=$a python scripts/decode_ab.py qwen2-57b-a14b 1 2 2>&1 | tail -1 | sed "s/^/async=$a /"
  HAP_GEMV_ASYNC=$a python scripts/decode_ab.py mixtral-8x7b 1 2 2>&1 | tail -1 | sed "s/^/async=$a /"
done; done
