for T in 1 4 8 16 32 64 128 256 512 1024; do
for m in 1024 0; do HAP_ROUTER_WIDE_MAXT=$m timeout 60 python scripts/router_decode_bench.py $T; done
done
