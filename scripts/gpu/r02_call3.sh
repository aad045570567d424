set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_boundary_peer_gpu.py tests/test_ep_peer_gpu.py tests/test_peer_allreduce_gpu.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/peer_tests.txt
cat gpurun_out/peer_tests.txt
bash scripts/gpu/attn_sweep.sh > gpurun_out/attn_ab2.txt 2>&1
cat gpurun_out/attn_ab2.txt
bash scripts/gpu/r02_gemm_l2.sh > /dev/null 2>&1
cat gpurun_out/gemm_l2_sweep.txt
