for rep in 1 2; do for c in 0 1; do
  HAP_CAPTURE_WARM_STREAM=$c python scripts/decode_ab.py qwen2-57b-a14b 1 2 64 2>&1 | tail -1 | sed "s/^/warm_stream=$c /"
  HAP_CAPTURE_WARM_STREAM=$c python scripts/decode_ab.py mixtral-8x7b 1 2 64 2>&1 | tail -1 | sed "s/^/warm_stream=$c /"
done; done
