mkdir -p gpurun_out
O=gpurun_out/sanitizer_detail.txt
: > $O
echo "## synccheck attn_prefill" >> $O
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "test_attn_prefill" -p no:cacheprovider >> $O 2>&1
echo "## racecheck one pair GEMM" >> $O
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 6 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "test_grouped_gemm_swiglu_ragged" -p no:cacheprovider >> $O 2>&1
tail -c 20000 $O
