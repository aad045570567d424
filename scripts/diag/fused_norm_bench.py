"""Decode attention prologue in isolation: rmsnorm + QKV (two launches) vs the
fused hap_rmsnorm_gemm_qkv_rope, 1-2 rows, weights streamed from HBM (an L2
flush precedes every call; its time alone is subtracted).  CUDA graphs, events.
  python scripts/diag/fused_norm_bench.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_2508_19373_b200 import ops

dev = "cuda"
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            flush.zero_()
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best


for name, K, nq, nkv, has_bias in (("qwen2-57b", 3584, 28, 4, True), ("mixtral", 4096, 32, 8, False)):
    d = 128
    N = (nq + 2 * nkv) * d
    w = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
    lnw = torch.ones(K, device=dev, dtype=torch.bfloat16)
    bias = torch.zeros(N, device=dev, dtype=torch.bfloat16) if has_bias else None
    t0 = graph_time(lambda: None)
    for M in (1, 2):
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        pos = torch.full((M,), 2047, device=dev, dtype=torch.int32)
        hn = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        two = graph_time(lambda: ops.gemm_qkv_rope(ops.rmsnorm(x, lnw, 1e-6, out=hn), w, pos, nq + nkv, d, 1e6,
                                                   bias=bias, out=out)) - t0
        norm = graph_time(lambda: ops.rmsnorm(x, lnw, 1e-6, out=hn)) - t0
        qkv = graph_time(lambda: ops.gemm_qkv_rope(hn, w, pos, nq + nkv, d, 1e6, bias=bias, out=out)) - t0
        fused = graph_time(lambda: ops.rmsnorm_qkv_rope(x, lnw, 1e-6, w, pos, nq + nkv, d, 1e6, bias=bias,
                                                        out=out)) - t0
        print(f"{name} M={M}: norm {norm:.1f} us, qkv {qkv:.1f} us, norm+qkv {two:.1f} us, fused {fused:.1f} us "
              f"({N * K * 2 / 1e6:.1f} MB weights)")
