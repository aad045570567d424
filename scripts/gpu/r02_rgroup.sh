for gsz in 8 4 8 4; do for T in 1 8; do HAP_ROUTER_GROUP=$gsz timeout 60 python scripts/router_decode_bench.py $T; done; done
HAP_ROUTER_GROUP=4 timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k router 2>&1 | tail -2
