"""Clock / power of the Mixtral expert gate/up GEMM in a long loop (dev
diagnostic): python scripts/diag/gemm_power.py [seconds].  Run with and without
HAP_GEMM_NOLOAD=1 (stages complete without TMA loads: tensor work alone) to see
how much of the power-capped clock the operand traffic costs."""
import os
import statistics
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import pynvml
import torch

from paper_2508_19373_b200 import ops

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
which = sys.argv[2] if len(sys.argv) > 2 else "gate_up"
E, h, I, rows = 8, 4096, 14336, 32768
x = torch.randn(rows, h, device="cuda").to(torch.bfloat16)
w13 = (torch.randn(E, 2 * I, h, device="cuda") * 0.02).to(torch.bfloat16)
seg = torch.arange(0, rows + 1, rows // E, device="cuda", dtype=torch.int32)
H = torch.empty(rows, I, device="cuda", dtype=torch.bfloat16)
hw = ops.swiglu_half_width(I)
w2 = (torch.randn(E, h, I, device="cuda") * 0.02).to(torch.bfloat16)
Y = torch.empty(rows, h, device="cuda", dtype=torch.bfloat16)
ops.grouped_gemm(x, w13, E, seg, H, swiglu_half=hw)
if which == "down":
    fn = lambda: ops.grouped_gemm(H, w2, E, seg, Y)  # noqa: E731
else:
    fn = lambda: ops.grouped_gemm(x, w13, E, seg, H, swiglu_half=hw)  # noqa: E731
for _ in range(5):
    fn()
torch.cuda.synchronize()
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hdl) / 1e3))
        time.sleep(0.02)


th = threading.Thread(target=sampler)
th.start()
n = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
s.record()
while time.time() - t0 < secs:
    for _ in range(20):
        fn()
    n += 20
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
stop.set()
th.join()
ms = s.elapsed_time(e) / n
late = samples[len(samples) // 3:]
flops = 2 * rows * 2 * I * h if which == "gate_up" else 2 * rows * I * h
print(f"{which} noload={os.environ.get('HAP_GEMM_NOLOAD', '0')}: {ms:.3f} ms/GEMM = {flops / ms / 1e9:.0f} TF/s, "
      f"SM clock median {statistics.median(c for c, _ in late):.0f} MHz, power median "
      f"{statistics.median(p for _, p in late):.0f} W ({len(late)} samples)")
