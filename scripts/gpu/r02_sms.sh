for i in 1 2; do
for c in "0 0" "48 100" "64 84" "74 74" "36 112" "100 48"; do
set -- $c
TAG="sh=$1 ro=$2" HAP_SHARED_SMS=$1 HAP_ROUTED_SMS=$2 timeout 300 python scripts/decode_half.py qwen2-57b-a14b 1
TAG="sh=$1 ro=$2" HAP_SHARED_SMS=$1 HAP_ROUTED_SMS=$2 timeout 300 python scripts/decode_half.py qwen2-57b-a14b 8
done
done
