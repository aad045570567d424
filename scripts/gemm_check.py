"""Time the tcgen05 grouped GEMM on the Mixtral expert shapes (dev script).

HAP_GEMM_CTA_PAIR=0 selects the 1-CTA variant for A/B comparison."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


dev = "cuda"
E, M_e, h, I = 8, 4096, 4096, 14336
seg = torch.arange(0, (E + 1) * M_e, M_e, dtype=torch.int32, device=dev)
A = torch.randn(E * M_e, h, device=dev).bfloat16()
W13 = (torch.randn(E * 2 * I, h, device=dev) * 0.02).bfloat16()
H = torch.empty(E * M_e, I, device=dev, dtype=torch.bfloat16)
ms = timed(lambda: ops.grouped_gemm(A, W13, E, seg, H, swiglu_half=128))
print(f"gate/up grouped (8 x 4096 x 28672 x 4096): {ms:.3f} ms  {2 * E * M_e * 2 * I * h / ms / 1e9:.1f} TFLOP/s")
W2 = (torch.randn(E * h, I, device=dev) * 0.02).bfloat16()
Y = torch.empty(E * M_e, h, device=dev, dtype=torch.bfloat16)
ms = timed(lambda: ops.grouped_gemm(H, W2, E, seg, Y))
print(f"down grouped (8 x 4096 x 4096 x 14336): {ms:.3f} ms  {2 * E * M_e * I * h / ms / 1e9:.1f} TFLOP/s")
X = torch.randn(16384, h, device=dev).bfloat16()
Wqkv = (torch.randn(6144, h, device=dev) * 0.02).bfloat16()
pos = torch.arange(2048, device=dev, dtype=torch.int32).repeat(8)
ms = timed(lambda: ops.gemm_qkv_rope(X, Wqkv, pos, 40, 128, 1e6))
print(f"qkv+rope (16384 x 6144 x 4096): {ms:.3f} ms  {2 * 16384 * 6144 * h / ms / 1e9:.1f} TFLOP/s")
Wo = (torch.randn(h, h, device=dev) * 0.02).bfloat16()
ms = timed(lambda: ops.gemm(X, Wo, residual=X))
print(f"o-proj (16384 x 4096 x 4096): {ms:.3f} ms  {2 * 16384 * h * h / ms / 1e9:.1f} TFLOP/s")
# decode-shaped: 16 rows per expert
segd = torch.arange(0, (E + 1) * 16, 16, dtype=torch.int32, device=dev)
Ad = torch.randn(E * 16, h, device=dev).bfloat16()
Hd = torch.empty(E * 16, I, device=dev, dtype=torch.bfloat16)
ms = timed(lambda: ops.grouped_gemm(Ad, W13, E, segd, Hd, swiglu_half=128))
print(f"decode gate/up (8 x 16 rows): {ms * 1e3:.1f} us  {E * 2 * I * h * 2 / ms / 1e9:.0f} GB/s weights")
