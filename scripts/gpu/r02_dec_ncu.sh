mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 1 -c 1 -f -o /tmp/dec python scripts/profile_decode.py mixtral-8x7b 64 3 > gpurun_out/dec_ncu.log 2>&1
ncu -i /tmp/dec.ncu-rep --page raw --csv > gpurun_out/dec_raw.csv 2>/dev/null
ncu -i /tmp/dec.ncu-rep --page details --csv > gpurun_out/dec_details.csv 2>/dev/null
ncu -i /tmp/dec.ncu-rep --page source --csv > gpurun_out/dec_source.csv 2>/dev/null
ls -la gpurun_out/dec_*
