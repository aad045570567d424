# One-box evidence pass: GPU suite, smoke, bench line, ncu launch list + full-set capture of one prefill block.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt
ls -la MEASURED_PEAKS.json >> gpurun_out/gpu_info.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_block.csv python scripts/profile_block.py 2 2 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -f -o gpurun_out/full_block python scripts/profile_block.py 1 0 > gpurun_out/ncu_full.log 2>&1
tail -c 1500 gpurun_out/bench.json
cat gpurun_out/pytest_gpu.txt | tail -5
cat gpurun_out/smoke.txt | tail -2
