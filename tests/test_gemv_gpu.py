"""The opt-in decode GEMV path of the GEMM entry points (gemm.cu gemv_kernel,
HAP_GEMV=2) against a torch fp32 reference of the same op: plain, bias +
residual, RoPE-QKV, SwiGLU, grouped SwiGLU / down with empty experts, 1-8
activation rows.  The mode is read once per process, so the checks run in a
child pytest with HAP_GEMV=2 (tolerance 1e-2 relative, bf16 output)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
INNER = os.environ.get("HAP_GEMV") == "2"
dev = "cuda"


def test_gemv_path_in_child_process():
    if INNER:
        pytest.skip("inner run")
    env = dict(os.environ, HAP_GEMV="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", str(Path(__file__)), "-k", "inner"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def r(*s, std=1.0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(*s, device=dev, generator=g) * std).to(torch.bfloat16)


def rope_ref(y, pos, n_heads, d, theta):
    T = y.shape[0]
    yh = y[:, : n_heads * d].view(T, n_heads, d)
    half = d // 2
    inv = 1.0 / theta ** (torch.arange(half, device=dev, dtype=torch.float64) * 2 / d)
    ang = pos.double()[:, None] * inv[None]
    c, s = ang.cos().float()[:, None], ang.sin().float()[:, None]
    x1, x2 = yh[..., :half], yh[..., half:]
    out = y.clone()
    out[:, : n_heads * d] = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1).reshape(T, -1)
    return out


@pytest.mark.skipif(not INNER, reason="runs in the HAP_GEMV=2 child")
@pytest.mark.parametrize("M", [1, 3, 8])
def test_inner_gemv_plain_bias_residual(M):
    from paper_2508_19373_b200 import ops

    a, w, b, res = r(M, 1024, seed=1), r(768, 1024, std=0.03, seed=2), r(768, seed=3), r(M, 768, seed=4)
    got = ops.gemm(a, w, bias=b, residual=res)
    ref = a.float() @ w.float().t() + b.float() + res.float()
    assert rel(got, ref) < 1e-2
    got = ops.gemm(a, w)
    assert rel(got, a.float() @ w.float().t()) < 1e-2


@pytest.mark.skipif(not INNER, reason="runs in the HAP_GEMV=2 child")
@pytest.mark.parametrize("M", [1, 5])
def test_inner_gemv_qkv_rope(M):
    from paper_2508_19373_b200 import ops

    nq, nkv, d, h = 8, 2, 128, 1024
    a, w, b = r(M, h, seed=5), r((nq + 2 * nkv) * d, h, std=0.03, seed=6), r((nq + 2 * nkv) * d, seed=7)
    pos = torch.randint(0, 4096, (M,), device=dev, dtype=torch.int32)
    got = ops.gemm_qkv_rope(a, w, pos, nq + nkv, d, 1e6, bias=b)
    ref = rope_ref(a.float() @ w.float().t() + b.float(), pos, nq + nkv, d, 1e6)
    assert rel(got, ref) < 1e-2


@pytest.mark.skipif(not INNER, reason="runs in the HAP_GEMV=2 child")
@pytest.mark.parametrize("M", [1, 8])
def test_inner_gemv_swiglu_and_grouped(M):
    from paper_2508_19373_b200 import ops
    from paper_2508_19373_b200.weights import interleave_gate_up

    h, inter, E = 512, 704, 6
    hw = ops.swiglu_half_width(inter)
    a = r(M, h, seed=8)
    w1, w3 = r(E, inter, h, std=0.04, seed=9), r(E, inter, h, std=0.04, seed=11)
    w13 = interleave_gate_up(w1, w3, hw)
    w2 = r(E, h, inter, std=0.04, seed=10)

    def swiglu(x, e):
        g, u = x.float() @ w1[e].float().t(), x.float() @ w3[e].float().t()
        return torch.nn.functional.silu(g) * u

    got = ops.gemm(a, w13[0], swiglu_half=hw)  # dense SwiGLU on expert 0
    assert rel(got, swiglu(a, 0)) < 1e-2
    # grouped: rows split over experts 1 and 4, the others empty
    cut = M // 2
    seg = torch.tensor([0, 0, cut, cut, cut, M, M], device=dev, dtype=torch.int32)
    H = torch.empty(M, inter, device=dev, dtype=torch.bfloat16)
    ops.grouped_gemm(a, w13, E, seg, H, swiglu_half=hw)
    Y = torch.empty(M, h, device=dev, dtype=torch.bfloat16)
    ops.grouped_gemm(H, w2, E, seg, Y)
    for e, (lo, hi) in ((1, (0, cut)), (4, (cut, M))):
        if hi <= lo:
            continue
        assert rel(H[lo:hi], swiglu(a[lo:hi], e)) < 1e-2
        assert rel(Y[lo:hi], H[lo:hi].float() @ w2[e].float().t()) < 1e-2


@pytest.mark.parametrize("M", [1, 2, 3, 9])
@pytest.mark.parametrize("dims", [(3584, 28, 4, True), (4096, 32, 8, False)], ids=["qwen2-57b", "mixtral"])
def test_fused_norm_qkv_matches_two_launches(M, dims):
    """hap_rmsnorm_gemm_qkv_rope (default mode: the GEMV stages the normalised
    rows itself at 1-2 rows, two launches otherwise) is bit-identical to
    hap_rmsnorm + hap_gemm_qkv_rope, and the rows it normalises equal
    hap_rmsnorm's output bit for bit (checked through the projection)."""
    if INNER:
        pytest.skip("default GEMV mode only")
    from paper_2508_19373_b200 import ops

    K, nq, nkv, has_bias = dims
    d = 128
    N = (nq + 2 * nkv) * d
    x = r(M, K, seed=M)
    lnw = (1.0 + 0.05 * r(K, seed=7).float()).to(torch.bfloat16)
    w = r(N, K, std=0.02, seed=3)
    bias = r(N, std=0.1, seed=4) if has_bias else None
    pos = torch.arange(100, 100 + M, device=dev, dtype=torch.int32) * 7
    want = ops.gemm_qkv_rope(ops.rmsnorm(x, lnw, 1e-6), w, pos, nq + nkv, d, 1e6, bias=bias)
    got = ops.rmsnorm_qkv_rope(x, lnw, 1e-6, w, pos, nq + nkv, d, 1e6, bias=bias)
    torch.cuda.synchronize()
    assert torch.equal(got, want), (M, dims, rel(got, want))


def test_fused_norm_decode_block_bit_identical():
    """The executor's opt-in fused decode prologue (HAP_FUSED_NORM=1) leaves the
    block's decode output and routing bit-identical."""
    if INNER:
        pytest.skip("default GEMV mode only")
    from paper_2508_19373_b200 import executor as E
    from paper_2508_19373_b200.config import get_config, scaled
    from paper_2508_19373_b200.layout import PlanDegrees

    cfg = scaled(get_config("qwen2-57b-a14b"), hidden=1024, n_q_heads=8, n_kv_heads=2, inter=512)
    blk = E.HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
    prev = E._FUSED_NORM
    try:
        for B in (1, 2, 5):
            torch.manual_seed(B)
            cache = E.KVCache.empty(B, cfg.n_kv_heads, 256, cfg.head_dim, dev, random=True)
            pos = torch.full((B,), 200, device=dev, dtype=torch.int32)
            x = r(B, cfg.hidden, seed=B)
            res = {}
            for f in (False, True):
                E._FUSED_NORM = f
                res[f] = (blk.forward(x, "decode", B, kv_cache=cache, positions=pos).clone(),
                          blk.last_routing[0].clone())
            assert torch.equal(res[False][0], res[True][0]) and torch.equal(res[False][1], res[True][1]), B
    finally:
        E._FUSED_NORM = prev

