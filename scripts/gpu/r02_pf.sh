for i in 1 2; do
for c in "0 0" "32 0" "64 0" "96 0" "64 1"; do
set -- $c
HAP_L2_PREFETCH_MB=$1 HAP_L2_PREFETCH_LAST=$2 timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 64 | sed "s/^/pf=$1 last=$2 /"
HAP_L2_PREFETCH_MB=$1 HAP_L2_PREFETCH_LAST=$2 timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 64 | sed "s/^/pf=$1 last=$2 /"
done
done
