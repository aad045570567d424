set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_boundary_peer_gpu.py tests/test_ep_peer_gpu.py tests/test_peer_allreduce_gpu.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/peer_tests.txt
cat gpurun_out/peer_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qwen2_b1.csv python scripts/profile_decode.py qwen2-57b-a14b 1 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mixtral_b64.csv python scripts/profile_decode.py mixtral-8x7b 64 2 > /dev/null 2>&1
timeout 900 python scripts/bench_configs.py gpurun_out/configs.json > gpurun_out/configs.log 2>&1
tail -12 gpurun_out/configs.log
