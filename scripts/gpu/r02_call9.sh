set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py tests/test_paged_kv_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/tests9.txt
cat gpurun_out/tests9.txt
for f in 1 0 1 0; do HAP_GEMM_FUSED_REDUCE=$f timeout 600 python scripts/bench_configs.py gpurun_out/configs_f$f.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/configs_f$f.json'))
print('fused=$f', [(r['workload'].split(' block ')[0][:12]+' '+r['workload'].split(' block ')[1], round(r['ms_per_step']*1e3,1)) for r in d['rows'] if 'decode' in r['workload']])"; done
timeout 300 python scripts/measure_reshard.py gpurun_out/reshard_measure.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/reshard_measure.json'))
for r in d['rows']: print(r['switch'], round(r['pack_ms'],3), round(r['unpack_ms'],3), round(r['transfer_ms_at_nvlink5'],3))"
