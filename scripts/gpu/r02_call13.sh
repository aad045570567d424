set -x
mkdir -p gpurun_out
timeout 3000 python scripts/calibrate.py > gpurun_out/r02_calibrate.log 2>&1
tail -8 gpurun_out/r02_calibrate.log
timeout 1500 python scripts/e2e_model.py --out gpurun_out/r02_e2e_model.json > gpurun_out/e2e.log 2>&1
tail -30 gpurun_out/e2e.log
