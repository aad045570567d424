mkdir -p gpurun_out
O=gpurun_out/sanitizer_detail2.txt
: > $O
for e in 0 1; do HAP_ATTN_EMU=0 timeout 60 python scripts/attn_bench.py >> $O 2>&1; done
echo "## synccheck kernels + block" >> $O
timeout 900 compute-sanitizer --tool synccheck --print-limit 4 python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py -m gpu -q -x -k "not full_size and not sweep and not 8x22b" -p no:cacheprovider 2>&1 | grep -v "Host Frame" | tail -40 >> $O
echo "## racecheck kernels (verbose)" >> $O
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest tests/test_kernels_gpu.py -m gpu -v -x -k "not full_size" -p no:cacheprovider 2>&1 | grep -v "Host Frame" | grep -B2 -A8 "Race reported\|RACECHECK SUMMARY" | head -60 >> $O
cat $O
