"""Child process for tests/test_gemv_gpu.py: dense 1-2-row GEMV outputs (store,
bias + residual, RoPE-QKV, SwiGLU, fused norm + QKV) hashed, so two processes
with different kernel-selection environments can be compared bit for bit."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

dev = "cuda"


def r(*s, std=1.0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(*s, device=dev, generator=g) * std).to(torch.bfloat16)


h = hashlib.sha256()
for M in (1, 2):
    for K, N in ((3584, 4608), (4096, 6144), (1024, 512)):
        x = r(M, K, seed=M + K)
        w = r(N, K, std=0.02, seed=N)
        res = r(M, N, seed=5)
        bias = r(N, std=0.1, seed=6)
        outs = [ops.gemm(x, w), ops.gemm(x, w, bias=bias, residual=res)]
        pos = torch.arange(M, device=dev, dtype=torch.int32) * 131 + 7
        outs.append(ops.gemm_qkv_rope(x, w, pos, N // 128, 128, 1e6, bias=bias))
        lnw = (1.0 + 0.05 * r(K, seed=9).float()).to(torch.bfloat16)
        outs.append(ops.rmsnorm_qkv_rope(x, lnw, 1e-6, w, pos, N // 128, 128, 1e6, bias=bias))
        outs.append(ops.gemm(x, w, swiglu_half=64))
        torch.cuda.synchronize()
        for o in outs:
            h.update(o.contiguous().view(torch.int16).cpu().numpy().tobytes())
print(h.hexdigest())
