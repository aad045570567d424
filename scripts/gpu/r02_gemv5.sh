for v in 0 1 0 1; do
HAP_GEMV=$v timeout 300 ncu --graph-profiling graph --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv python scripts/profile_decode.py qwen2-57b-a14b 1 6 graph 2>/dev/null | grep -i duration | awk -v v=$v -F'","' '{print "gemv=" v, $NF}'
done
