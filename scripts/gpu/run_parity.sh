# headline-config parity tests (round 2) + the fp32-accumulate GEMM check
nproc
timeout 1500 python -m pytest tests/test_block_gpu.py tests/test_kernels_gpu.py -m gpu -q -k "full_size or fp32 or block_tiny or geometry or shared_expert or decode_step" -s --durations=15 2>&1 | grep -E "row-relative|per-element|flips|passed|failed|Error|assert" > gpurun_out/r02_parity.txt
cat gpurun_out/r02_parity.txt
