"""Graph-replayed decode step of one preset block at several batches (A/B helper, dev script):
python scripts/decode_ab.py <preset> B1 [B2 ...]  -> 'B=..: .. us' per batch."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch

from bench_configs import timed
from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
from paper_2508_19373_b200.layout import PlanDegrees

torch.manual_seed(0)  # same routing in every process
cfg = get_config(sys.argv[1])
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
out = []
for B in map(int, sys.argv[2:]):
    cache = KVCache.empty(B, cfg.n_kv_heads, 2048, cfg.head_dim, "cuda", random=True)
    pos = torch.full((B,), 2047, device="cuda", dtype=torch.int32)
    x = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
    graph, _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
    out.append(f"B={B}: {timed(graph.replay, steps=100, warmup=20) * 1e3:.1f}us")
print(f"gemv={os.environ.get('HAP_GEMV', '1')} pdl={os.environ.get('HAP_PDL', '0')} {sys.argv[1]} " + ", ".join(out))
