# Attention A/B (HAP_ATTN_EMU), GPU suite, bench, ncu launch list + selective full-set captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt
for e in 0 1 0 1; do HAP_ATTN_EMU=$e timeout 60 python scripts/attn_bench.py; done > gpurun_out/attn_ab.txt 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attn" 2>&1 | tail -3 >> gpurun_out/attn_ab.txt
cat gpurun_out/attn_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 2>&1 | tail -20 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_block.csv python scripts/profile_block.py 2 2 > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -f -o /tmp/full_block python scripts/profile_block.py 1 0 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/full_block.ncu-rep --page raw --csv > gpurun_out/full_block_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pair -c 1 -f -o gpurun_out/attn_full python scripts/profile_block.py 1 0 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out; du -sh gpurun_out
tail -c 2500 gpurun_out/bench.json
tail -4 gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/smoke.txt
