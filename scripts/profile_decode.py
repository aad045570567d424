"""One decode step of a preset block at batch B (kv 2048) a few times, for ncu
launch lists: python scripts/profile_decode.py <preset> <B> [n_steps] [graph]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
from paper_2508_19373_b200.layout import PlanDegrees

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "qwen2-57b-a14b")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
cache = KVCache.empty(B, cfg.n_kv_heads, 2048, cfg.head_dim, "cuda", random=True)
pos = torch.full((B,), 2047, device="cuda", dtype=torch.int32)
x = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
if graph:
    g, _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
    for _ in range(n):
        g.replay()
else:
    for _ in range(n):
        blk.forward(x, "decode", B, kv_cache=cache, positions=pos, max_position=2047)
torch.cuda.synchronize()
print("done")
