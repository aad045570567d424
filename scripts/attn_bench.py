"""Time hap_attn_prefill on the Mixtral-8x7B prefill shape (dev script)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2508_19373_b200 import ops
B, S, nq, nkv, d = 8, 2048, 32, 8, 128
qkv = torch.randn(B * S, (nq + 2 * nkv) * d, device="cuda").to(torch.bfloat16)
out = torch.empty(B * S, nq * d, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.attn_prefill(qkv, nq, nkv, d, B, S, out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.attn_prefill(qkv, nq, nkv, d, B, S, out)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
fl = 4 * B * S * S * nq * d / 2  # causal useful
print(f"attn prefill {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s (causal useful)")
