for i in 1 2; do
for c in 0 50 60 66 74 84 96; do
HAP_SHARED_SMS=$c timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 512 | sed "s/^/sh=$c /"
done
done
