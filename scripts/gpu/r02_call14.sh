set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:router -c 2 -f -o gpurun_out/router_full python scripts/profile_block.py 1 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:router_group -c 1 -f -o gpurun_out/router_group_full python scripts/profile_decode.py qwen2-57b-a14b 1 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
