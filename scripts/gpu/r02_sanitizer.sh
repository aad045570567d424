# compute-sanitizer over the shipped kernels at HEAD: memcheck + synccheck on the kernel and
# block test files (small shapes), racecheck on the kernel tests; one log for profiles/.
mkdir -p gpurun_out
L=gpurun_out/compute_sanitizer.txt
git_rev=$(cat .git_rev 2>/dev/null || echo unknown)
echo "# HEAD $git_rev; $(date -u)" > $L
SEL="not full_size and not sweep and not 8x22b"
for tool in memcheck synccheck; do
  echo "## $tool: tests/test_kernels_gpu.py tests/test_block_gpu.py tests/test_gemv_gpu.py tests/test_paged_kv_gpu.py tests/test_copy2d_gpu.py -k '$SEL'" >> $L
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_kernels_gpu.py tests/test_block_gpu.py tests/test_gemv_gpu.py tests/test_paged_kv_gpu.py tests/test_copy2d_gpu.py -m gpu -q -x -k "$SEL" -p no:cacheprovider 2>&1 | tail -8 >> $L
done
echo "## racecheck: tests/test_kernels_gpu.py tests/test_gemv_gpu.py" >> $L
timeout 2400 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_kernels_gpu.py tests/test_gemv_gpu.py -m gpu -q -x -k "$SEL" -p no:cacheprovider 2>&1 | tail -8 >> $L
echo "## memcheck: smoke()" >> $L
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4 >> $L
cat $L
