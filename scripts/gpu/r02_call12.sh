set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "router or qwen" 2>&1 | tail -4 > gpurun_out/tests12.txt
cat gpurun_out/tests12.txt
for i in 1 2; do timeout 300 python scripts/profile_decode.py qwen2-57b-a14b 1 3 > /dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qwen2_b1.csv python scripts/profile_decode.py qwen2-57b-a14b 1 2 > /dev/null 2>&1
timeout 900 python scripts/bench_configs.py gpurun_out/configs12.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/configs12.json'))
for r in d['rows']: print(r['workload'], round(r['ms_per_step'],3))"
timeout 1500 python scripts/e2e_model.py --out gpurun_out/r02_e2e_model.json > gpurun_out/e2e.log 2>&1
tail -45 gpurun_out/e2e.log
