mkdir -p gpurun_out
for v in 0 1; do
HAP_GEMV=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gemv_dec_$v.csv python scripts/profile_decode.py qwen2-57b-a14b 1 3 > /dev/null 2>&1
done
ls -la gpurun_out
