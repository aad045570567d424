set -x
mkdir -p gpurun_out
for t in 1 2 1 2; do HAP_ROUTER_TPL=$t timeout 60 python scripts/router_bench.py; done > gpurun_out/router_ab.txt 2>&1
cat gpurun_out/router_ab.txt
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "router or tiny or mixtral" 2>&1 | tail -3
