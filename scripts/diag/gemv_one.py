"""One dense decode GEMV launch (Mixtral QKV, 1 row) for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_2508_19373_b200 import ops

K, N = 4096, 6144
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
x = torch.randn(1, K, device="cuda").to(torch.bfloat16)
pos = torch.full((1,), 2047, device="cuda", dtype=torch.int32)
for _ in range(3):
    ops.gemm_qkv_rope(x, w, pos, 48, 128, 1e6)
torch.cuda.synchronize()
