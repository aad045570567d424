"""Diagnostic: where the end-to-end error of the full-size Mixtral prefill parity check comes from."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import conftest  # noqa: F401  (sys.path for baseline/_ref)
import test_block_gpu as T
from oracle import moe_block as O
from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock
from paper_2508_19373_b200.layout import PlanDegrees
from paper_2508_19373_b200.weights import synthetic_weights

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b")
B, S = 8, 2048
W = synthetic_weights(cfg, "cuda", seed=0)
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
blk.capture = {}
g = torch.Generator(device="cuda"); g.manual_seed(123)
x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
out = blk.forward(x, "prefill", B, S); torch.cuda.synchronize()
h1 = T.np32(blk.capture["h1"]); hn = T.np32(blk.capture["hn_s"]); got = T.np32(out)
idx = blk.last_routing[0].cpu().numpy(); tw = blk.capture["topk_w"].cpu().numpy()
spec = T.oracle_spec(cfg)
Wa = T._np_weights(W, T._ATTN_KEYS)
P = 2048
h1r = O.attention_module(spec, Wa, T.np32(x[:P]), 1, bf16_mirror=True)["h1"]
hnr = O.bf16_round(O.rmsnorm(h1r, Wa["ln2"], spec.rms_eps).astype(np.float32))
lgr = O.router_logits(hnr, T.np32(W["router"]))
oir, owr = O.router_topk(lgr, cfg.top_k, cfg.norm_topk_prob)
lgg = O.router_logits(hn[:P], T.np32(W["router"]))
print("h1 elem err", T.elem_rel_err(h1[:P], h1r), "h1 maxnorm err", T.rel_err_rows(h1[:P], h1r))
print("hn elem err", T.elem_rel_err(hn[:P], hnr))
print("logit max abs diff", np.abs(lgg - lgr).max(), "logit std", lgr.std())
print("topk weight max abs diff", np.abs(tw[:P] - owr).max())
agree = (np.sort(idx[:P], 1) == np.sort(oir, 1)).all(1)
m = O.topk_margin(lgr, cfg.top_k)
print("flips", (~agree).sum(), "margins", np.sort(m[~agree])[-5:] if (~agree).any() else None)
s = np.linspace(0, P - 1, 128).astype(np.int64)
s = s[agree[s]]
moe_g = T._moe_ref(cfg, W, hn[s], (idx[s], tw[s]))
moe_r = T._moe_ref(cfg, W, hnr[s], (oir[s], owr[s]))
gpu_moe = got[s] - h1[s]
def rep(name, a, b):
    e = np.abs(a - b) / np.maximum(np.abs(b), np.sqrt(np.mean(b * b, -1, keepdims=True)))
    i = np.unravel_index(np.argmax(e), e.shape)
    print(f"{name}: elem {e.max():.3e} at {i} got {a[i]:.4f} ref {b[i]:.4f}; maxnorm {np.abs(a-b).max()/np.abs(b).max():.3e}; p99.99 {np.quantile(e, 0.9999):.3e}")
rep("moe(hn_gpu) vs moe(hn_ref)", moe_g, moe_r)
rep("gpu moe vs moe(hn_gpu)", gpu_moe, moe_g)
rep("out vs h1_gpu+moe(hn_gpu)", got[s], h1[s] + moe_g)
rep("out vs h1_ref+moe(hn_ref)", got[s], h1r[s] + moe_r)
rep("h1_gpu vs h1_ref", h1[s], h1r[s])
print("rms out", np.sqrt(np.mean(got[s] ** 2)), "rms moe", np.sqrt(np.mean(moe_r ** 2)))
