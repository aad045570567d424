"""Mixtral-8x7B expert GEMMs in isolation (32768 routed rows, 4096 per expert):
time gate/up and down with CUDA events (dev script for the L2 raster / cache
hint experiments; run under ncu for DRAM bytes).  Env knobs are read by the
library: HAP_GEMM_RASTER_MB, HAP_GEMM_RASTER_N, HAP_GEMM_HINT."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

E, h, I, rows = 8, 4096, 14336, 32768
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(rows, h, device="cuda", generator=g).to(torch.bfloat16)
w13 = (torch.randn(E, 2 * I, h, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
w2 = (torch.randn(E, h, I, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
seg = torch.arange(0, rows + 1, rows // E, device="cuda", dtype=torch.int32)
if os.environ.get("SWEEP_RAGGED") == "1":  # segment sizes of a random top-2 routing (multinomial), not 4096 each
    cnt = torch.bincount(torch.randint(0, E, (rows,), generator=torch.Generator().manual_seed(3)), minlength=E)
    seg = torch.zeros(E + 1, dtype=torch.int32)
    seg[1:] = torch.cumsum(cnt, 0)
    seg = seg.to("cuda")
hw = ops.swiglu_half_width(I)
H = torch.empty(rows, I, device="cuda", dtype=torch.bfloat16)
Y = torch.empty(rows, h, device="cuda", dtype=torch.bfloat16)
res = {}
for name, fn in (("gate_up", lambda: ops.grouped_gemm(x, w13, E, seg, H, swiglu_half=hw)),
                 ("down", lambda: ops.grouped_gemm(H, w2, E, seg, Y))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    res[name] = s.elapsed_time(e) / reps
tag = " ".join(f"{k}={os.environ[k]}" for k in ("HAP_GEMM_RASTER_MB", "HAP_GEMM_RASTER_N", "HAP_GEMM_HINT")
               if k in os.environ) or "default"
print(f"{tag}: gate_up {res['gate_up']:.3f} ms ({2*rows*2*I*h/res['gate_up']/1e9:.0f} TF/s), "
      f"down {res['down']:.3f} ms ({2*rows*I*h/res['down']/1e9:.0f} TF/s)", flush=True)
