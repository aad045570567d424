for v in 0 1 0 1; do HAP_PDL=$v timeout 600 python scripts/bench_configs.py /tmp/c$v.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('/tmp/c$v.json'))
print('pdl=$v', [(r['workload'].split(' block ')[1], round(r['ms_per_step']*1e3,1)) for r in d['rows']])"; done
