for f in 1 0; do HAP_FUSED_NORM=$f timeout 600 python -m pytest tests/test_block_gpu.py -m gpu -q -s -k "full_size_mixtral_decode or qwen2_57b_decode_sweep" 2>&1 | grep -E "flips|passed|failed|assert" | sed "s/^/fused=$f /"; done > gpurun_out/seed_check.txt
cat gpurun_out/seed_check.txt
