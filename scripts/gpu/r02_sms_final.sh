# shared-expert SM budget sweep on the final code (Qwen2-57B decode; HAP_SHARED_SMS, default 74 = half)
for rep in 1 2; do for sms in 64 74 84 96; do
  HAP_SHARED_SMS=$sms python scripts/decode_ab.py qwen2-57b-a14b 1 2 8 64 2>&1 | tail -1 | sed "s/^/sms=$sms /"
done; done
