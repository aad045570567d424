set -x
mkdir -p gpurun_out
HAP_DIST_BACKEND=gloo timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/gloo_n4.json 2> gpurun_out/gloo_n4.err
tail -c 3000 gpurun_out/gloo_n4.json; grep -v "^\s*$" gpurun_out/gloo_n4.err | grep -iv "warn\|omp_num\|\*\*\*" | tail -8
