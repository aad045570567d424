for r in 0 1; do
  echo "== ragged=$r"
  SWEEP_RAGGED=$r timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 6 --csv python scripts/gemm_l2_sweep.py 1 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
