"""Time hap_attn_prefill on the Mixtral-8x7B prefill shape, causal and non-causal (dev script).
HAP_ATTN_EMU=0|1 selects all exponentials on the SFU | one pair in four on the FMA pipe."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2508_19373_b200 import ops
B, S, nq, nkv, d = 8, 2048, 32, 8, 128
qkv = torch.randn(B * S, (nq + 2 * nkv) * d, device="cuda").to(torch.bfloat16)
out = torch.empty(B * S, nq * d, device="cuda", dtype=torch.bfloat16)
res = []
for causal in (True, False):
    for _ in range(3):
        ops.attn_prefill(qkv, nq, nkv, d, B, S, out, causal=causal)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        ops.attn_prefill(qkv, nq, nkv, d, B, S, out, causal=causal)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    fl = 4 * B * S * S * nq * d / (2 if causal else 1)  # causal: useful half
    res.append(f"{'causal' if causal else 'full'} {ms*1e3:.1f} us {fl/ms/1e9:.0f} TF/s")
print(f"emu={os.environ.get("HAP_ATTN_EMU", "default")}: " + "; ".join(res))
