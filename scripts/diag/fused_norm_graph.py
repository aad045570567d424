"""One process, one block: the decode step with the attention norm fused into
the QKV launch vs separate (executor._FUSED_NORM toggled), eager outputs
compared bit for bit, then both CUDA graphs replayed alternately.
  python scripts/diag/fused_norm_graph.py <preset> B"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from bench_configs import timed
from paper_2508_19373_b200 import executor as E
from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.layout import PlanDegrees

torch.manual_seed(0)
cfg = get_config(sys.argv[1])
B = int(sys.argv[2])
blk = E.HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
cache = E.KVCache.empty(B, cfg.n_kv_heads, 2048, cfg.head_dim, "cuda", random=True)
pos = torch.full((B,), 2047, device="cuda", dtype=torch.int32)
x = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
outs, routes, graphs = {}, {}, {}
for f in (False, True):
    E._FUSED_NORM = f
    outs[f] = blk.forward(x, "decode", B, kv_cache=cache, positions=pos).clone()
    routes[f] = blk.last_routing[0].clone()
    graphs[f], _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
torch.cuda.synchronize()
print("outputs bit-identical:", torch.equal(outs[False], outs[True]), "routing identical:",
      torch.equal(routes[False], routes[True]))
for rep in range(3):
    print(" ".join(f"fused={int(f)} {timed(graphs[f].replay, steps=100, warmup=20) * 1e3:.1f}us" for f in (False, True)))
