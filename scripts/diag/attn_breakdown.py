"""Diagnostic: attention-module error chain at full size (qkv -> attention -> o-proj -> h1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import conftest  # noqa: F401
import test_block_gpu as T
from oracle import moe_block as O
from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock
from paper_2508_19373_b200.layout import PlanDegrees
from paper_2508_19373_b200.weights import synthetic_weights

name, B, S, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = get_config(name)
W = synthetic_weights(cfg, "cuda", seed=0)
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None, weights=W)
blk.capture = {}
g = torch.Generator(device="cuda"); g.manual_seed(123)
x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
out = blk.forward(x, "prefill", B, S); torch.cuda.synchronize()
cap = {k: T.np32(v[:P]) for k, v in blk.capture.items() if k in ("qkv", "attn", "h1")}
spec = T.oracle_spec(cfg)
Wa = T._np_weights(W, T._ATTN_KEYS)
d, Hq, Hkv = cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
xs = T.np32(x[:P])
def rep(name, a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    fl = np.sqrt(np.mean(b * b, -1, keepdims=True))
    e = np.abs(a - b) / np.maximum(np.abs(b), fl)
    i = np.unravel_index(np.argmax(e), e.shape)
    print(f"{name}: elem {e.max():.3e} at {i} got {a[i]:.5f} ref {b[i]:.5f} rowrms {fl[i[0],0]:.4f}; row-rel {T.row_rel_err(a,b):.3e}; p99.9 {np.quantile(e,0.999):.3e}")
# qkv: oracle from x (bf16 mirrored), rope applied
xn = O.bf16_round(O.rmsnorm(xs, Wa["ln1"], spec.rms_eps).astype(np.float32)).astype(np.float64)
q = xn @ Wa["wq"].astype(np.float64).T; k = xn @ Wa["wk"].astype(np.float64).T; v = xn @ Wa["wv"].astype(np.float64).T
pos = np.arange(P)
qr = O.rope(q.reshape(P, Hq, d), pos, spec.rope_theta).reshape(P, -1)
kr = O.rope(k.reshape(P, Hkv, d), pos, spec.rope_theta).reshape(P, -1)
rep("qkv (GPU vs oracle, GEMM+RoPE)", cap["qkv"], np.concatenate([qr, kr, v], 1))
# attention on the GPU's own q,k,v
gq = cap["qkv"][:, :Hq * d].reshape(P, Hq, d); gk = cap["qkv"][:, Hq * d:(Hq + Hkv) * d].reshape(P, Hkv, d)
gv = cap["qkv"][:, (Hq + Hkv) * d:].reshape(P, Hkv, d)
att = O.attention(gq, gk, gv).reshape(P, -1)
rep("attn (GPU vs oracle on GPU qkv)", cap["attn"], att)
# o-proj on GPU attention output
h1v = xs.astype(np.float64) + cap["attn"].astype(np.float64) @ Wa["wo"].astype(np.float64).T
rep("h1 (GPU vs oracle o-proj on GPU attn)", cap["h1"], h1v)
h1r = O.attention_module(spec, Wa, xs, 1, bf16_mirror=True)["h1"]
rep("h1 (GPU vs oracle end to end)", cap["h1"], h1r)
rep("h1 oracle-on-GPU-attn vs oracle e2e", h1v, h1r)
attr = O.bf16_round(O.attention(O.bf16_round(qr.astype(np.float32)).reshape(P,Hq,d), O.bf16_round(kr.astype(np.float32)).reshape(P,Hkv,d), O.bf16_round(v.astype(np.float32)).reshape(P,Hkv,d)).reshape(P,-1).astype(np.float32))
rep("attn GPU vs oracle e2e attn", cap["attn"], attr)
# per-row scale of the attention output vs position
rms_att = np.sqrt(np.mean(att ** 2, -1))
print("attn row rms at pos 0,1,10,100,P-1:", rms_att[[0, 1, 10, 100, P - 1]])
