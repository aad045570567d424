"""Time hap_attn_decode on Mixtral decode B=64, kv 2048 (dev script)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2508_19373_b200 import ops
B, L, nq, nkv, d = 64, 2048, 32, 8, 128
qkv = torch.randn(B, (nq + 2 * nkv) * d, device="cuda").to(torch.bfloat16)
kc = torch.randn(B, nkv, L, d, device="cuda").to(torch.bfloat16)
vc = torch.randn(B, nkv, L, d, device="cuda").to(torch.bfloat16)
pos = torch.full((B,), L - 1, device="cuda", dtype=torch.int32)
out = torch.empty(B, nq * d, device="cuda", dtype=torch.bfloat16)
ws = torch.empty(ops.attn_decode_workspace_bytes(B, nq, d, L), device="cuda", dtype=torch.uint8)
for _ in range(3):
    ops.attn_decode(qkv, kc, vc, pos, nq, nkv, d, out, ws)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    ops.attn_decode(qkv, kc, vc, pos, nq, nkv, d, out, ws)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
byts = 2 * B * nkv * L * d * 2
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} decode attn {ms*1e3:.1f} us  {byts/ms/1e9:.0f} GB/s")
