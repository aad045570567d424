# Final evidence on the final code: GPU suite, smoke, bench (ours + reference arm), ncu launch list +
# full-set capture (raw CSV only; the .ncu-rep is too large to bring back), per-config table.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -20 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_block.csv python scripts/profile_block.py 2 2 > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -f -o /tmp/full_block python scripts/profile_block.py 1 0 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/full_block.ncu-rep --page raw --csv > gpurun_out/full_block_raw.csv 2>/dev/null
timeout 900 python scripts/bench_configs.py gpurun_out/configs.json > gpurun_out/configs.log 2>&1
tail -c 1200 gpurun_out/bench.json
tail -c 600 gpurun_out/bench_ref.json
tail -4 gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/smoke.txt
