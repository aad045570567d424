for i in 1 2; do
for c in "0 0" "74 74" "74 0" "0 74" "68 80" "80 68" "70 70" "60 60"; do
set -- $c
TAG="sh=$1 ro=$2" HAP_SHARED_SMS=$1 HAP_ROUTED_SMS=$2 timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 | sed "s/^/sh=$1 ro=$2 /"
done
done
