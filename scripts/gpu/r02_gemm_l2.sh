# L2 raster / cache-hint sweep of the Mixtral expert GEMMs: event timings, then DRAM bytes under ncu.
mkdir -p gpurun_out
O=gpurun_out/gemm_l2_sweep.txt
: > $O
V=("" "HAP_GEMM_HINT=LF" "HAP_GEMM_HINT=FL" "HAP_GEMM_HINT=LN" "HAP_GEMM_HINT=NL" "HAP_GEMM_RASTER_MB=24" "HAP_GEMM_RASTER_MB=96" "HAP_GEMM_RASTER_MB=160" "HAP_GEMM_RASTER_N=1" "HAP_GEMM_RASTER_N=1 HAP_GEMM_RASTER_MB=24" "HAP_GEMM_RASTER_N=1 HAP_GEMM_RASTER_MB=96")
for v in "${V[@]}"; do env $v timeout 120 python scripts/gemm_l2_sweep.py 10 >> $O 2>&1; done
for v in "${V[@]}"; do
  echo "== ncu $v" >> $O
  env $v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:grouped_gemm -c 6 --csv python scripts/gemm_l2_sweep.py 1 2>/dev/null | grep -E "dram__bytes|lts__t_sector_hit|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tail -24 >> $O
done
cat $O
