"""Time hap_router_topk at a decode shape (Qwen2-57B: h=3584, 64 experts + shared gate, top-8), T tokens;
dev script for the wide-router A/B (HAP_ROUTER_GROUP)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1
h, E, k = 3584, 64, 8
x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
w = (torch.randn(E + 1, h, device="cuda") * 0.02).to(torch.bfloat16)
idx = torch.empty(T, k, device="cuda", dtype=torch.int32)
tw = torch.empty(T, k, device="cuda", dtype=torch.float32)
sg = torch.empty(T, device="cuda", dtype=torch.float32)
fn = lambda: ops.router_topk(x, w, E, k, False, True, idx, tw, sg)  # noqa: E731
for _ in range(5):
    fn()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        fn()
g.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    g.replay()
e.record()
torch.cuda.synchronize()
print(f"group={os.environ.get('HAP_ROUTER_GROUP', '4')} wide_maxt={os.environ.get('HAP_ROUTER_WIDE_MAXT', '-')} T={T}: {s.elapsed_time(e) / 200 * 1e3:.1f} us per router call (graph)")
