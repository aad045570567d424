set -x
mkdir -p gpurun_out
HAP_GEMM_MC=1 timeout 120 python scripts/gemm_l2_sweep.py 3 > gpurun_out/mc_first.txt 2>&1; echo "rc=$?" >> gpurun_out/mc_first.txt
cat gpurun_out/mc_first.txt
if grep -q "rc=0" gpurun_out/mc_first.txt; then
  HAP_GEMM_MC=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "gemm" 2>&1 | tail -3
  HAP_GEMM_MC=1 timeout 600 python -m pytest tests/test_block_gpu.py -m gpu -q -x -k "tiny or mixtral_geometry or qwen_shared or full_size_mixtral_prefill" 2>&1 | tail -3
  for v in 0 1 0 1; do HAP_GEMM_MC=$v timeout 120 python scripts/gemm_l2_sweep.py 10; done
  for v in 0 1 0 1; do HAP_GEMM_MC=$v timeout 120 python scripts/diag/gemm_power.py 4 | sed "s/^/mc=$v /"; done
fi
