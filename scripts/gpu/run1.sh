set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu_s1.txt
timeout 600 python bench.py > gpurun_out/r02_bench_s1.json 2> gpurun_out/r02_bench_s1.err
tail -c 3000 gpurun_out/r02_bench_s1.json
cat gpurun_out/r02_pytest_gpu_s1.txt
