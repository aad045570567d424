for v in 1 0 1 0; do HAP_GEMM_SNAKE=$v timeout 600 python bench.py --no-decode --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('snake=$v', round(d['ms_per_step'],3), round(d['kernels']['gate_up']['ms'],3), round(d['kernels']['down']['ms'],3), d['clocks']['sm_mhz'])"; done
