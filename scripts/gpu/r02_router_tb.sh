timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "router or qwen or decode" 2>&1 | tail -2
for T in 8 16 32 64 128 256 512 1024; do
for v in 0 1; do HAP_ROUTER_TB=$v timeout 60 python scripts/router_decode_bench.py $T | sed "s/^/tb=$v /"; done
done
for v in 0 1; do HAP_ROUTER_TB=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 16 64 256 512 | sed "s/^/tb=$v /"; done
for v in 0 1; do HAP_ROUTER_TB=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 16 64 256 512 | sed "s/^/tb=$v /"; done
