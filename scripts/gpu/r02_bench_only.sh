mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info2.txt
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 900 python scripts/bench_configs.py gpurun_out/configs2.json > gpurun_out/configs2.log 2>&1
tail -c 400 gpurun_out/bench2.json
