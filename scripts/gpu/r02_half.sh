for i in 1 2; do
for g in 0 1; do
TAG=old HAP_GEMV=$g HAP_KERNELS_LIB=$PWD/ab_lib/old.so timeout 300 python scripts/decode_half.py qwen2-57b-a14b 1
TAG=new HAP_GEMV=$g timeout 300 python scripts/decode_half.py qwen2-57b-a14b 1
done
TAG=old HAP_KERNELS_LIB=$PWD/ab_lib/old.so timeout 300 python scripts/decode_half.py mixtral-8x7b 1
TAG=new timeout 300 python scripts/decode_half.py mixtral-8x7b 1
done
