"""Time hap_router_topk at the Mixtral-8x7B prefill shape (T=16384, h=4096, E=8, k=2), dev script for the
router A/B (HAP_ROUTER_TPL)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

T, h, E, k = 16384, 4096, 8, 2
x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
w = (torch.randn(E, h, device="cuda") * 0.02).to(torch.bfloat16)
idx = torch.empty(T, k, device="cuda", dtype=torch.int32)
tw = torch.empty(T, k, device="cuda", dtype=torch.float32)
for _ in range(3):
    ops.router_topk(x, w, E, k, True, False, idx, tw)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50):
    ops.router_topk(x, w, E, k, True, False, idx, tw)
e.record()
torch.cuda.synchronize()
us = s.elapsed_time(e) / 50 * 1e3
gbs = (T * h * 2 + E * h * 2 + T * k * 8) / (us * 1e-6) / 1e9
print(f"tpl={os.environ.get('HAP_ROUTER_TPL', 'default')}: {us:.1f} us = {gbs:.0f} GB/s")
