# full GPU suite, then the B200 recalibration (balanced + skewed routing)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r02_pytest_gpu.txt
cat gpurun_out/r02_pytest_gpu.txt
timeout 2400 python scripts/calibrate.py > gpurun_out/r02_calibrate.log 2>&1
tail -45 gpurun_out/r02_calibrate.log
