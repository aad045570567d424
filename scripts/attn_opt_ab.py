"""A/B of the optimistic softmax (HAP_ATTN_OPT) — run as two processes; this one
times hap_attn_prefill at the Mixtral prefill shape and saves the output for a
bit-identity check between the two modes."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

B, S, nq, nkv, d = 8, 2048, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(5)
qkv = torch.randn(B * S, (nq + 2 * nkv) * d, device="cuda", generator=g).to(torch.bfloat16)
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
    e.record()
    torch.cuda.synchronize()
    res.append(f"{'causal' if causal else 'full'} {s.elapsed_time(e) / 20 * 1e3:.1f} us")
    if causal:
        torch.save(out.cpu(), f"/tmp/attn_opt_{os.environ.get('HAP_ATTN_OPT', '1')}.pt")
print(f"opt={os.environ.get('HAP_ATTN_OPT', 'default')}: " + "; ".join(res))
