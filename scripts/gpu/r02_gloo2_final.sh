# multi-rank bench path on the final code, ranks sharing one B200 over gloo (code-path validation, not scaling):
# default line (NCCL-style collectives) and the opt-in --peer variant
mkdir -p gpurun_out
HAP_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 3 --warmup 3 --peer > gpurun_out/gloo_n2.json 2> gpurun_out/gloo_n2.err
echo "exit $?"
tail -1 gpurun_out/gloo_n2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('metric','value','n_gpus','ms_per_step')}); print(json.dumps(d.get('plans'))[:600]); print(json.dumps(d.get('hap_peer_exchanges'))[:400])"
grep -v "^\s*$" gpurun_out/gloo_n2.err | grep -iv "warn\|omp_num\|\*\*\*" | tail -5
