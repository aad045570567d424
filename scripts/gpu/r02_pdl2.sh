timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in 0 3 0 3; do HAP_PDL=$v timeout 300 python scripts/decode_ab.py qwen2-57b-a14b 1 8 64 512; HAP_PDL=$v timeout 300 python scripts/decode_ab.py mixtral-8x7b 1 64; done
for v in 0 3; do HAP_PDL=$v timeout 600 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pdl=$v prefill', d['ms_per_step'], 'decode', d.get('decode',{}).get('ms_per_step'))"; done
