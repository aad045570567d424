for v in 0 1; do
HAP_GEMV=$v timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/gemv_warm_$v.csv python scripts/profile_decode.py qwen2-57b-a14b 1 4 graph > /dev/null 2>&1
done
