mkdir -p gpurun_out
for rep in 1 2; do for f in 0 1; do
  HAP_FUSED_NORM=$f python scripts/decode_half.py mixtral-8x7b 1 2>&1 | tail -1 | sed "s/^/fused=$f mixtral B=1 /"
  HAP_FUSED_NORM=$f python scripts/decode_half.py qwen2-57b-a14b 1 2>&1 | tail -1 | sed "s/^/fused=$f qwen B=1 /"
done; done > gpurun_out/fused_half.txt
cat gpurun_out/fused_half.txt
