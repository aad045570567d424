set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "gemm or rope" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_block_gpu.py tests/test_paged_kv_gpu.py -m gpu -q -x -k "decode or model or tiny or paged" 2>&1 | tail -15
for v in 1 0 1 0; do HAP_GEMV=$v timeout 600 python scripts/bench_configs.py /tmp/c$v.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('/tmp/c$v.json'))
print('gemv=$v', [(r['workload'].split(' block ')[1], round(r['ms_per_step']*1e3,1)) for r in d['rows'] if 'decode' in r['workload']])"; done
