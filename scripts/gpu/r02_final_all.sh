# final evidence on the final code: everything in r02_final.sh, then the sanitizer pass
bash scripts/gpu/r02_final.sh
bash scripts/gpu/r02_sanitizer.sh > /dev/null 2>&1
tail -30 gpurun_out/compute_sanitizer.txt
