"""Run the Mixtral-8x7B block (prefill 8x2048, then decode B=64 kv 2048) a few
times for ncu captures: python scripts/profile_block.py [n_prefill] [n_decode]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200.config import get_config
from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
from paper_2508_19373_b200.layout import PlanDegrees

n_p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_d = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = get_config(sys.argv[3] if len(sys.argv) > 3 else "mixtral-8x7b")
blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
x = torch.randn(8 * 2048, cfg.hidden, device="cuda").to(torch.bfloat16)
for _ in range(n_p):
    blk.forward(x, "prefill", 8, 2048)
cache = KVCache.empty(64, cfg.n_kv_heads, 2048, cfg.head_dim, "cuda", random=True)
pos = torch.full((64,), 2047, device="cuda", dtype=torch.int32)
xd = torch.randn(64, cfg.hidden, device="cuda").to(torch.bfloat16)
for _ in range(n_d):
    blk.forward(xd, "decode", 64, kv_cache=cache, positions=pos, max_position=2047)
torch.cuda.synchronize()
print("done")
