set -x
mkdir -p gpurun_out
git_rev=$(cat .git_rev 2>/dev/null)
timeout 600 python -m pytest tests/test_paged_kv_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "paged or model or decode" 2>&1 | tail -15 > gpurun_out/tests6.txt
cat gpurun_out/tests6.txt
bash scripts/gpu/r02_sanitizer.sh > /dev/null 2>&1
cat gpurun_out/compute_sanitizer.txt
