for v in 0 1 0 1; do HAP_GEMM_SNAKE=$v timeout 120 python scripts/diag/gemm_power.py 4 down | sed "s/^/snake=$v /"; done
for v in 0 1; do
  echo "== snake=$v"
  HAP_GEMM_SNAKE=$v timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 6 --csv python scripts/gemm_l2_sweep.py 1 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tail -4
done
HAP_GEMM_SNAKE=1 timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k gemm 2>&1 | tail -2
