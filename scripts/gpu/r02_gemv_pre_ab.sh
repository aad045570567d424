# GEMV first-group prefetch before the activation staging: same-box A/B against the previous build (libhap_base.so)
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export HAP_KERNELS_LIB=$PWD/paper_2508_19373_b200/libhap_base.so; else unset HAP_KERNELS_LIB; fi
    python scripts/diag/fused_norm_bench.py 2>&1 | tail -4 | grep -o "^[a-z0-9-]* M=[12]: .*qkv [0-9.]* us" | sed "s/^/$lib /" | tr '\n' ';'; echo
    python scripts/decode_ab.py qwen2-57b-a14b 1 2 2>&1 | tail -1 | sed "s/^/$lib /"
    python scripts/decode_ab.py mixtral-8x7b 1 2 2>&1 | tail -1 | sed "s/^/$lib /"
  done
done
