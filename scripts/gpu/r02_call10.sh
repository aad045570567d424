set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "positions_outside" 2>&1 | tail -40 > gpurun_out/t10a.txt
cat gpurun_out/t10a.txt
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py tests/test_paged_kv_gpu.py -m gpu -q 2>&1 | tail -8 > gpurun_out/tests10.txt
cat gpurun_out/tests10.txt
for f in 1 0 1 0; do HAP_GEMM_FUSED_REDUCE=$f timeout 600 python scripts/bench_configs.py gpurun_out/configs_f$f.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/configs_f$f.json'))
print('fused=$f', [(r['workload'].split(' block ')[1], round(r['ms_per_step']*1e3,1)) for r in d['rows'] if 'decode' in r['workload']])"; done
