for v in 0 3 4; do
  echo "== noload=$v"
  HAP_GEMM_NOLOAD=$v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 3 --csv python scripts/gemm_l2_sweep.py 1 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tail -3
done
