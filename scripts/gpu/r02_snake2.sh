for mb in 24 48 96 160 48; do HAP_GEMM_RASTER_MB=$mb timeout 120 python scripts/diag/gemm_power.py 4 down | sed "s/^/mb=$mb /"; done
for mb in 24 48 96; do HAP_GEMM_RASTER_MB=$mb timeout 120 python scripts/diag/gemm_power.py 4 gate_up | sed "s/^/mb=$mb /"; done
