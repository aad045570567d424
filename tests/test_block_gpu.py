"""Block-level parity on one B200: the executor's full MoE block vs the CPU oracle.

Parity definition:
  1. routing indices bit-exact — the oracle's fixed-order router applied to
     the GPU's own normalised router input gives identical top-k;
  2. permutation bit-exact — (dst_of_row, seg) equal the oracle's stable
     counting sort of those indices;
  3. block output within bf16 tolerance: max |gpu - oracle| / max |oracle|
     <= 2e-2 against the oracle run with bf16 rounding at the executor's
     storage points, over tokens whose routing agrees (a bf16 rounding
     difference in the router *input* can legitimately flip a near-tie);
     at least 99% of tokens must agree, and every token that disagrees must
     be a near-tie of the oracle's own logits (``near_tie_only``);
  4. fp32 quantities (router logits, routing weights) within 1e-4.

At the BASELINE sizes (``check_full_size``):
  * module level (oracle experts on the GPU's router input and routing): the
    block output per element, |gpu - ref| <= 2e-2 * max(|ref|, rms(ref row))
    (``elem_rel_err``);
  * end to end from the same x (oracle attention module -> oracle router on
    the oracle's own router input -> oracle experts) on whole sequences: per
    row max|gpu - ref| / max|ref| <= 2e-2 (``row_rel_err``), and per element
    within 2e-2 plus the oracle's own spread: the oracle run on the GPU's
    (bf16) h1 and router input differs from the oracle run end to end by up to
    3-5e-2 per element, because a one-ulp difference of a bf16 h1 / router
    input element (different fp32 accumulation order in attention) moves the
    fp64 expert MLP output (profiles/r02_parity_breakdown.txt).  By the
    triangle inequality this bound is the module-level check carried to the
    end-to-end reference; the row bound is the independent one.
"""

import numpy as np
import pytest
import torch

from oracle import moe_block as O

pytestmark = pytest.mark.gpu


def np32(t):
    return t.detach().float().cpu().numpy()


def oracle_spec(cfg):
    return O.BlockSpec(hidden=cfg.hidden, n_q_heads=cfg.n_q_heads, n_kv_heads=cfg.n_kv_heads,
                       head_dim=cfg.head_dim, n_experts=cfg.n_experts, top_k=cfg.top_k, inter=cfg.inter,
                       n_shared=cfg.n_shared, norm_topk_prob=cfg.norm_topk_prob, qkv_bias=cfg.qkv_bias,
                       rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)


def run_block(cfg, batch, seq, seed=0):
    from paper_2508_19373_b200.executor import HapMoEBlock
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    W = synthetic_weights(cfg, "cuda", seed=seed)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
    blk.capture = {}
    g = torch.Generator(device="cuda")
    g.manual_seed(123)
    x = torch.randn(batch * seq, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    out = blk.forward(x, "prefill", batch, seq)
    torch.cuda.synchronize()
    Wn = {k: np32(v) for k, v in W.items()}
    return blk, x, out, Wn


def check_block(cfg, batch, seq):
    blk, x, out, Wn = run_block(cfg, batch, seq)
    spec = oracle_spec(cfg)
    idx, dst, seg = (t.cpu().numpy() for t in blk.last_routing)
    hn = np32(blk.capture["hn_s"])
    # (1) routing bit-exact on the GPU's own router input
    logits = O.router_logits(hn, Wn["router"])
    oi, ow = O.router_topk(logits, cfg.top_k, cfg.norm_topk_prob)
    assert np.array_equal(idx, oi)
    assert np.abs(blk.capture["topk_w"].cpu().numpy() - ow).max() < 1e-4
    # (2) permutation bit-exact
    od, os_ = O.permute_index(oi.reshape(-1), cfg.n_experts)
    assert np.array_equal(dst, od) and np.array_equal(seg, os_)
    # (3) block output vs the independent oracle forward
    ref = O.block_forward(spec, Wn, np32(x), batch, bf16_mirror=True)
    agree = near_tie_only(idx, ref["topk_idx"], ref["logits"], cfg.top_k)
    assert agree.mean() >= 0.99, f"routing agreement {agree.mean():.4f}"
    got = np32(out)
    err = rel_err_rows(got[agree], ref["out"][agree])
    assert err <= 2e-2, err
    # the attention module alone (h1) is routing independent
    assert rel_err_rows(np32(blk.capture["h1"]), ref["h1"]) <= 2e-2
    return err


def rel_err_rows(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def row_rel_err(got, ref):
    """max over rows of max|got - ref| / max|ref| (each row judged on its own scale)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref).max(-1) / np.abs(ref).max(-1)))


def check_e2e(got, ref, what, via=None):
    """End-to-end bound (see the module docstring).  via: the oracle evaluated
    on the GPU's own intermediates (h1, router input, routing); its distance
    to ref is the oracle's own spread, allowed on top of 2e-2 per element."""
    r, e = row_rel_err(got, ref), elem_rel_err(got, ref)
    spread = elem_rel_err(via, ref) if via is not None else 0.0
    print(f"{what}: row-relative {r:.3e}, per-element {e:.3e} (oracle spread {spread:.3e})")
    assert r <= 2e-2 and e <= 2e-2 + spread, (what, r, e, spread)


def elem_rel_err(got, ref):
    """max over elements of |got - ref| / max(|ref|, rms of the ref row): a
    per-element relative error whose denominator is floored at the row's RMS
    (an element near zero is judged against the row's scale)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    floor = np.sqrt(np.mean(ref * ref, axis=-1, keepdims=True))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), floor)))


# a bf16 rounding of the router input moves fp32 logits by ~|x|*|w|*2^-9*sqrt(h);
# routing may legitimately differ only where the oracle's k-th / (k+1)-th logit
# gap is below this (the logits have std ~1.3 at init std 0.02)
NEAR_TIE = 5e-2


def near_tie_only(idx_gpu, idx_ref, logits_ref, top_k):
    """Tokens whose top-k sets differ must be near-ties of the reference logits."""
    agree = (np.sort(idx_gpu, 1) == np.sort(idx_ref, 1)).all(1)
    margin = O.topk_margin(logits_ref, top_k)
    if (~agree).any():
        print(f"routing flips: {(~agree).sum()} of {agree.size}, max oracle margin {margin[~agree].max():.3e}")
    bad = (~agree) & (margin > NEAR_TIE)
    assert not bad.any(), f"routing differs on {bad.sum()} tokens with margin > {NEAR_TIE}: {margin[bad][:5]}"
    return agree


def test_block_tiny():
    from paper_2508_19373_b200.config import get_config

    check_block(get_config("tiny"), 4, 128)


def test_block_mixtral_geometry_small():
    """Mixtral-8x7B head/expert geometry with a reduced intermediate size and hidden."""
    from paper_2508_19373_b200.config import get_config, scaled

    cfg = scaled(get_config("mixtral-8x7b"), hidden=1024, n_q_heads=8, n_kv_heads=2, inter=1792)
    check_block(cfg, 2, 256)


def test_block_qwen_shared_expert():
    from paper_2508_19373_b200.config import get_config, scaled

    cfg = scaled(get_config("qwen1.5-moe-a2.7b"), hidden=1024, n_q_heads=8, n_kv_heads=8)
    check_block(cfg, 2, 128)


def test_block_qwen2_57b_geometry_small():
    from paper_2508_19373_b200.config import get_config, scaled

    cfg = scaled(get_config("qwen2-57b-a14b"), hidden=1792, n_q_heads=14, n_kv_heads=2)
    check_block(cfg, 2, 64)


def test_decode_step_matches_oracle():
    from paper_2508_19373_b200.config import get_config
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = get_config("tiny")
    W = synthetic_weights(cfg, "cuda", seed=3)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
    B, Lmax = 6, 300
    cache = KVCache.empty(B, cfg.n_kv_heads, Lmax, cfg.head_dim, "cuda", random=True)
    k0, v0 = np32(cache.k), np32(cache.v)
    pos = torch.tensor([0, 5, 64, 255, 256, 299], device="cuda", dtype=torch.int32)
    x = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
    out = blk.forward(x, "decode", B, kv_cache=cache, positions=pos)
    torch.cuda.synchronize()
    Wn = {k: np32(v) for k, v in W.items()}
    ref = O.decode_forward(oracle_spec(cfg), Wn, np32(x), k0, v0, pos.cpu().numpy())
    idx = blk.last_routing[0].cpu().numpy()
    agree = (np.sort(ref["topk_idx"], 1) == np.sort(idx, 1)).all(1)
    got = np32(out)
    assert agree.sum() >= B - 1
    assert rel_err_rows(got[agree], ref["out"][agree]) <= 3e-2


def test_model_prefill_then_decode_matches_oracle():
    """Two stacked tiny blocks: prefill fills the KV caches (checked against
    the oracle's post-RoPE k/v), then graph-replayed decode steps append and
    attend; every output vs the chained oracle (bf16 tolerance)."""
    from paper_2508_19373_b200.config import get_config
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.model import HapModel
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = get_config("tiny")
    L, B, S, steps, max_len = 2, 2, 64, 3, 80
    model = HapModel(cfg, PlanDegrees(1, 1, 1, 1), None, n_layers=L, seed=5)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    caches = model.new_caches(B, max_len)
    out = model.prefill(x, B, S, caches)
    spec = oracle_spec(cfg)
    Ws = [{k: np32(v) for k, v in synthetic_weights(cfg, "cuda", seed=5 * 1000 + l).items()} for l in range(L)]
    h = np32(x)
    ocaches = []
    for l in range(L):
        res = O.block_forward(spec, Ws[l], h, B, bf16_mirror=True)
        ocaches.append(list(O.caches_from_prefill(res, B, max_len)))
        if l == 0:  # cache fill: post-RoPE k and v of every prompt token
            assert rel_err_rows(np32(caches[0].k)[:, :, :S], ocaches[0][0][:, :, :S]) < 2e-2
            assert rel_err_rows(np32(caches[0].v)[:, :, :S], ocaches[0][1][:, :, :S]) < 2e-2
        h = res["out"]
    assert rel_err_rows(np32(out), h) < 3e-2
    pos = torch.full((B,), S, device="cuda", dtype=torch.int32)
    xd = torch.empty(B, cfg.hidden, device="cuda", dtype=torch.bfloat16)
    graph, gout = model.capture_decode(xd, B, caches, pos)
    for step in range(steps):
        xs = torch.randn(B, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
        xd.copy_(xs)
        graph.replay()
        torch.cuda.synchronize()
        hp = np32(xs)
        p = np.full(B, S + step)
        for l in range(L):
            res = O.decode_forward(spec, Ws[l], hp, ocaches[l][0], ocaches[l][1], p)
            O.append_kv(ocaches[l][0], ocaches[l][1], res, p)
            hp = res["out"]
        assert rel_err_rows(np32(gout), hp) < 3e-2, step
        pos += 1


def test_forward_host_streams_chunks_identically():
    """Host-buffer prefill (pipelined across calls, optional sequence chunks)
    gives bit-identical output to one device forward over the whole batch."""
    from paper_2508_19373_b200.config import get_config, scaled

    cfg = scaled(get_config("mixtral-8x7b"), hidden=1024, n_q_heads=8, n_kv_heads=2, inter=1792)
    blk, x, out, _ = run_block(cfg, 4, 256)
    xh = x.cpu().pin_memory()
    for chunks in (1, 4, 2):
        oh = torch.zeros_like(xh).pin_memory()
        blk.forward_host(xh, oh, 4, 256, n_chunks=chunks)
        blk.host_sync()
        torch.cuda.synchronize()
        assert torch.equal(oh, out.cpu())


def test_forward_host_pipelines_successive_batches():
    """Three batches queued back to back (H2D of i+1 and D2H of i overlap the
    forward of i): every output equals its own device forward."""
    from paper_2508_19373_b200.config import get_config, scaled

    cfg = scaled(get_config("mixtral-8x7b"), hidden=1024, n_q_heads=8, n_kv_heads=2, inter=1792)
    blk, _, _, _ = run_block(cfg, 2, 256)
    xs = [torch.randn(512, cfg.hidden, device="cuda").to(torch.bfloat16) for _ in range(3)]
    refs = [blk.forward(x, "prefill", 2, 256).cpu() for x in xs]
    hs = [x.cpu().pin_memory() for x in xs]
    outs = [torch.zeros_like(h).pin_memory() for h in hs]
    for h, o in zip(hs, outs):
        blk.forward_host(h, o, 2, 256)
    blk.host_sync()
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)


# ---------------------------------------------------------------------------
# BASELINE.json configs 2-5 at their full sizes (N = 1 here; the multi-GPU
# plans are covered on gloo).  The checks, per config:
#   * routing bit-exact for EVERY token (oracle fixed-order router on the
#     GPU's own router input), routing weights within 1e-4, the permutation
#     bit-exact for every row;
#   * expert module (sampled tokens): out == h1 + moe(hn) with the oracle's
#     fp64 experts on the GPU's hn and routing, per element within 2e-2;
#   * end to end from the same x on whole sequences (prefill: the first
#     min(S, 2048) tokens of sequence 0 — causal, so they depend only on
#     themselves; decode: up to 64 sequences): oracle attention module (bf16
#     rounding mirrored) -> oracle router on the oracle's own router input ->
#     oracle experts.  h1 per element within 2e-2; routing equal except on
#     near-ties of the oracle's logits; out per element within 2e-2 on tokens
#     whose routing agrees (>= 99 %).
class _LazyW(dict):
    """Oracle weight dict that pulls per-expert slices from the GPU on demand."""

    def __init__(self, W):
        super().__init__()
        self.W = W

    def __getitem__(self, k):
        t = self.W[k]
        if k in ("w1", "w2", "w3"):
            return _LazyExperts(t)
        return np32(t)


class _LazyExperts:
    def __init__(self, t):
        self.t = t

    def __getitem__(self, e):
        return np32(self.t[e])


def _np_weights(W, keys):
    return {k: np32(W[k]) for k in keys if k in W}


_ATTN_KEYS = ("ln1", "wq", "wk", "wv", "wo", "bq", "bk", "bv", "ln2")


def _moe_ref(cfg, W, hn, routing):
    return O.moe_forward(oracle_spec(cfg), _LazyW(W), hn, routing=routing)["moe"]


def _check_routing_all(cfg, blk, W):
    idx, dst, seg = (t.cpu().numpy() for t in blk.last_routing)
    od, os_ = O.permute_index(idx.reshape(-1), cfg.n_experts)
    assert np.array_equal(dst, od) and np.array_equal(seg, os_)
    hn = np32(blk.capture["hn_s"])
    oi, ow = O.router_topk(O.router_logits(hn, np32(W["router"])), cfg.top_k, cfg.norm_topk_prob)
    assert np.array_equal(idx, oi), f"routing differs on {(idx != oi).any(1).sum()} tokens"
    tw = blk.capture["topk_w"].cpu().numpy()
    assert np.abs(tw - ow).max() < 1e-4
    return idx, tw, hn


def check_full_size(cfg, batch, seq, n_sample=192, e2e_tokens=2048, n_e2e=128):
    from paper_2508_19373_b200.executor import HapMoEBlock
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    W = synthetic_weights(cfg, "cuda", seed=0)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
    blk.capture = {}
    g = torch.Generator(device="cuda")
    g.manual_seed(123)
    T = batch * seq
    x = torch.randn(T, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    out = blk.forward(x, "prefill", batch, seq)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    idx, tw, hn = _check_routing_all(cfg, blk, W)
    h1 = np32(blk.capture["h1"])
    cap_qkv, cap_attn = blk.capture["qkv"], blk.capture["attn"]
    got = np32(out)
    del blk
    # end to end from x: the first P tokens of sequence 0
    P = min(seq, e2e_tokens)
    spec = oracle_spec(cfg)
    Wa = _np_weights(W, _ATTN_KEYS)
    xs = np32(x[:P])
    h1_ref = O.attention_module(spec, Wa, xs, 1, bf16_mirror=True)["h1"]
    # module level: attention core on the GPU's own q/k/v, o-proj on the GPU's attention output
    d, Hq, Hkv = cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
    qkv, att = np32(cap_qkv[:P]), np32(cap_attn[:P])
    att_ref = O.attention(qkv[:, :Hq * d].reshape(P, Hq, d), qkv[:, Hq * d:(Hq + Hkv) * d].reshape(P, Hkv, d),
                          qkv[:, (Hq + Hkv) * d:].reshape(P, Hkv, d)).reshape(P, -1)
    err_att = elem_rel_err(att, att_ref)
    h1_via = xs.astype(np.float64) + att.astype(np.float64) @ Wa["wo"].astype(np.float64).T
    err_o = elem_rel_err(h1[:P], h1_via)
    print(f"{cfg.name} attention core (module level): per-element {err_att:.3e}; o-proj + residual {err_o:.3e}")
    assert err_att <= 2e-2 and err_o <= 2e-2, (err_att, err_o)
    check_e2e(h1[:P], h1_ref, f"{cfg.name} h1", via=h1_via)
    hn_ref = O.bf16_round(O.rmsnorm(h1_ref, Wa["ln2"], spec.rms_eps).astype(np.float32))
    lg_ref = O.router_logits(hn_ref, np32(W["router"]))
    oi_ref, ow_ref = O.router_topk(lg_ref, cfg.top_k, cfg.norm_topk_prob)
    agree = near_tie_only(idx[:P], oi_ref, lg_ref, cfg.top_k)
    assert agree.mean() >= 0.99, agree.mean()
    # one oracle expert pass over both samples: module level (GPU hn, GPU routing)
    # and end to end (oracle hn, oracle routing)
    # and end to end (oracle hn, oracle routing), plus the oracle on the GPU's
    # hn for the end-to-end tokens (the oracle's own spread)
    s_mod = np.linspace(0, T - 1, n_sample).astype(np.int64)
    s_e2e = np.linspace(0, P - 1, n_e2e).astype(np.int64)
    hn_all = np.concatenate([hn[s_mod], hn_ref[s_e2e], hn[s_e2e]])
    r_all = (np.concatenate([idx[s_mod], oi_ref[s_e2e], idx[s_e2e]]),
             np.concatenate([tw[s_mod], ow_ref[s_e2e], tw[s_e2e]]))
    moe = _moe_ref(cfg, W, hn_all, r_all)
    m_mod, m_e2e, m_via = moe[:n_sample], moe[n_sample:n_sample + n_e2e], moe[n_sample + n_e2e:]
    err_mod = elem_rel_err(got[s_mod], h1[s_mod] + m_mod)
    print(f"{cfg.name} out (module level): per-element {err_mod:.3e}")
    assert err_mod <= 2e-2, err_mod
    ok = agree[s_e2e]
    check_e2e(got[s_e2e][ok], h1_ref[s_e2e][ok] + m_e2e[ok], f"{cfg.name} out (end to end)",
              via=(h1[s_e2e] + m_via)[ok])


def test_full_size_mixtral_prefill():
    """BASELINE config 2 (the headline bench config): Mixtral-8x7B block, prefill 8 x 2048."""
    from paper_2508_19373_b200.config import get_config

    check_full_size(get_config("mixtral-8x7b"), 8, 2048)


def test_full_size_qwen15_moe_prefill():
    """BASELINE config 3 block (60 routed experts top-4 + 4 shared units, sigmoid-gated), prefill 8 x 2048."""
    from paper_2508_19373_b200.config import get_config

    check_full_size(get_config("qwen1.5-moe-a2.7b"), 8, 2048)


def test_full_size_mixtral_8x22b_prefill():
    """BASELINE config 5 block (h 6144, 48/8 heads, I 16384), prefill 16 x 4096 (T = 65536)."""
    from paper_2508_19373_b200.config import get_config

    check_full_size(get_config("mixtral-8x22b"), 16, 4096, n_sample=128, e2e_tokens=1024, n_e2e=96)


def check_full_size_decode(cfg, batch, L=2048, n_e2e=64):
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    W = synthetic_weights(cfg, "cuda", seed=0)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
    blk.capture = {}
    torch.manual_seed(11)  # the random cache must not depend on which tests ran before in this process
    cache = KVCache.empty(batch, cfg.n_kv_heads, L, cfg.head_dim, "cuda", random=True)
    pos = torch.full((batch,), L - 1, device="cuda", dtype=torch.int32)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn(batch, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    nb = min(batch, n_e2e)
    k0, v0 = np32(cache.k[:nb]), np32(cache.v[:nb])
    out = blk.forward(x, "decode", batch, kv_cache=cache, positions=pos)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    idx, tw, hn = _check_routing_all(cfg, blk, W)
    h1, got = np32(blk.capture["h1"]), np32(out)
    kn, vn = np32(cache.k[:nb, :, L - 1]), np32(cache.v[:nb, :, L - 1])
    # expert module on the GPU's hn and routing
    s = np.arange(nb)
    moe = _moe_ref(cfg, W, hn[s], (idx[s], tw[s]))
    err_mod = elem_rel_err(got[s], h1[s] + moe)
    print(f"{cfg.name} decode B={batch} out (module level): per-element {err_mod:.3e}")
    assert err_mod <= 2e-2, err_mod
    # end to end from x (oracle attention over cache + new token, oracle routing)
    ref = O.decode_forward(oracle_spec(cfg), _LazyW(W), np32(x[:nb]), k0, v0, pos[:nb].cpu().numpy())
    check_e2e(h1[:nb], ref["h1"], f"{cfg.name} decode B={batch} h1")
    # the new token's post-RoPE k and its v were appended at pos
    check_e2e(kn.reshape(nb, -1), ref["k"].reshape(nb, -1), "k appended")
    check_e2e(vn.reshape(nb, -1), ref["v"].reshape(nb, -1), "v appended")
    agree = near_tie_only(idx[:nb], ref["topk_idx"], ref["logits"], cfg.top_k)
    # every flip is a near-tie (asserted above); top-8 of 64 has many close gaps,
    # so bound their number rather than the fraction (one flip is 100 % at B=1)
    assert (~agree).sum() <= max(1, int(0.1 * nb)), (~agree).sum()
    if agree.any():
        check_e2e(got[:nb][agree], ref["out"][agree], f"{cfg.name} decode B={batch} out (end to end)",
                  via=(h1[s] + moe)[agree])


def test_full_size_mixtral_decode_b64():
    """BASELINE config 2, decode half: Mixtral-8x7B block, batch 64 at kv 2048."""
    from paper_2508_19373_b200.config import get_config

    check_full_size_decode(get_config("mixtral-8x7b"), 64)


@pytest.mark.parametrize("batch", [1, 8, 64, 512])
def test_full_size_qwen2_57b_decode_sweep(batch):
    """BASELINE config 4 block (64 experts top-8 + 8 shared units), decode at kv 2048 over the batch sweep."""
    from paper_2508_19373_b200.config import get_config

    check_full_size_decode(get_config("qwen2-57b-a14b"), batch)
