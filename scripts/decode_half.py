"""Decode step split for A/B work (dev script): graph-replayed time of the
whole block, of the attention half alone (experts stubbed out), and of the
expert half alone (attention stubbed): python scripts/decode_half.py <preset> B."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch

from bench_configs import timed
from paper_2508_19373_b200 import ops
from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
from paper_2508_19373_b200.layout import PlanDegrees

torch.manual_seed(0)  # same routing in every process
cfg = get_config(sys.argv[1])
B = int(sys.argv[2])
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
cache = KVCache.empty(B, cfg.n_kv_heads, 2048, cfg.head_dim, "cuda", random=True)
pos = torch.full((B,), 2047, device="cuda", dtype=torch.int32)
x = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
res = {}
g, _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
res["full"] = timed(g.replay, steps=100, warmup=20)
experts = blk._experts
blk._experts = lambda hn_s, residual, **kw: residual
g, _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
res["attn_half"] = timed(g.replay, steps=100, warmup=20)
blk._experts = experts
hn = ops.rmsnorm(x, blk.w.ln2, cfg.rms_eps)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        blk._experts(hn, x, res_row0=0, res_rows=B)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    blk._experts(hn, x, res_row0=0, res_rows=B)
res["expert_half"] = timed(g.replay, steps=100, warmup=20)
tag = os.environ.get("TAG", "")
print(f"{tag} gemv={os.environ.get('HAP_GEMV', '1')} {sys.argv[1]} B={B}: " +
      ", ".join(f"{k} {v * 1e3:.1f}us" for k, v in res.items()))
