set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reshard_gpu.py tests/test_boundary_peer_gpu.py tests/test_kernels_gpu.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/tests5.txt
cat gpurun_out/tests5.txt
timeout 600 python scripts/measure_reshard.py gpurun_out/reshard_measure.json > gpurun_out/reshard.log 2>&1
tail -30 gpurun_out/reshard.log
timeout 900 python scripts/bench_configs.py gpurun_out/configs.json > gpurun_out/configs.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/configs.json'))
for r in d['rows']: print(r['workload'], round(r['ms_per_step'],3), round(r.get('frac_of_hbm_peak', r.get('frac_of_sustained_bf16_peak',0)),3))"
HAP_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/gloo_n2.json 2> gpurun_out/gloo_n2.err
tail -c 1500 gpurun_out/gloo_n2.json; tail -5 gpurun_out/gloo_n2.err
