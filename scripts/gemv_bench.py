"""Decode-shape projections, tensor-core tiles vs the GEMV path (HAP_GEMV), dev script:
Qwen2-57B B=1 QKV (+RoPE), O (+residual), shared gate/up (SwiGLU) / down, routed gate/up / down."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200 import ops

h, nq, nkv, d, I, E, k, ns = 3584, 28, 4, 128, 2560, 64, 8, 8
dev = "cuda"
r = lambda *s: (torch.randn(*s, device=dev) * 0.02).to(torch.bfloat16)  # noqa: E731
M = int(os.environ.get("GEMV_ROWS", "1"))  # decode batch
x1 = r(M, h)
wqkv, bqkv = r((nq + 2 * nkv) * d, h), r((nq + 2 * nkv) * d)
pos = torch.full((M,), 2047, device=dev, dtype=torch.int32)
wo = r(h, nq * d)
attn = r(M, nq * d)
ws13, ws2 = r(2 * ns * I, h), r(h, ns * I)
w13, w2 = r(E, 2 * I, h), r(E, h, I)
xp = r(k, h)
seg = torch.zeros(E + 1, device=dev, dtype=torch.int32)
seg[1:] = torch.clamp(torch.arange(1, E + 1, device=dev), max=k).to(torch.int32)  # experts 0..7 one row each
H = torch.empty(k, I, device=dev, dtype=torch.bfloat16)
hw = ops.swiglu_half_width(I)
hws = ops.swiglu_half_width(ns * I)
def rot(make, nbytes):
    """Rotate over enough weight copies that the stream comes from HBM, not L2 (126 MB)."""
    n = max(1, -(-(256 << 20) // nbytes))
    fns = [make() for _ in range(n)]
    it = iter(range(1 << 30))
    return lambda: fns[next(it) % n]()


def copies(*ts):
    return [t.clone() for t in ts]


def mk_qkv():
    w, b = copies(wqkv, bqkv)
    return lambda: ops.gemm_qkv_rope(x1, w, pos, nq + nkv, d, 1e6, bias=b)


def mk_o():
    (w,) = copies(wo)
    return lambda: ops.gemm(attn, w, residual=x1)


def mk_sgu():
    (w,) = copies(ws13)
    return lambda: ops.gemm(x1, w, swiglu_half=hws)


hs = torch.empty(M, ns * I, device=dev, dtype=torch.bfloat16)


def mk_sd():
    (w,) = copies(ws2)
    return lambda: ops.gemm(hs, w)


cases = {
    "qkv_rope": rot(mk_qkv, wqkv.numel() * 2),
    "o_proj": rot(mk_o, wo.numel() * 2),
    "shared_gate_up": rot(mk_sgu, ws13.numel() * 2),
    "shared_down": rot(mk_sd, ws2.numel() * 2),
    "routed_gate_up": lambda: ops.grouped_gemm(xp, w13, E, seg, H, swiglu_half=hw),
    "routed_down": lambda: ops.grouped_gemm(H, w2, E, seg, torch.empty(k, h, device=dev, dtype=torch.bfloat16)),
}
out = []
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    out.append(f"{name} {s.elapsed_time(e) / 100 * 1e3:.1f}us")
print(f"M={M} gemv={os.environ.get('HAP_GEMV', '1')}: " + ", ".join(out))
