"""Worker for tests/test_reshard_gpu.py: ranks share cuda:0; the expert weights
live on the GPU and the reshard all-to-all is staged through gloo."""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(rank, world, port, cfg_kw, pairs, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.layout import PlanDegrees, RankLayout
    from paper_2508_19373_b200.transition import reshard_expert_weights
    from paper_2508_19373_b200.weights import pack_rank_weights, synthetic_weights

    cfg = BlockConfig(**cfg_kw)
    W = synthetic_weights(cfg, "cuda", seed=0)
    res = {}
    for (ti, ei), (tj, ej) in pairs:
        mk = lambda t, e: RankLayout(PlanDegrees(1, world, t, e, 1), rank, cfg.n_q_heads, cfg.n_kv_heads,  # noqa: E731
                                     cfg.n_experts, cfg.inter, cfg.n_shared)
        li, lj = mk(ti, ei), mk(tj, ej)
        wi = pack_rank_weights(cfg, W, li)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = reshard_expert_weights(cfg, wi, li, lj)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        want = pack_rank_weights(cfg, W, lj)
        ok = all((getattr(got, n) is None and getattr(want, n) is None) or torch.equal(getattr(got, n), getattr(want, n))
                 for n in ("w13", "w2", "ws13", "ws2"))
        ok = ok and got.w13.is_cuda and got.hw == want.hw and got.inter_local == want.inter_local
        res[f"{ti},{ei}->{tj},{ej}"] = {"ok": bool(ok), "seconds": dt}
    Path(f"{out_path}.{rank}").write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    a = json.loads(sys.argv[1])
    main(a["rank"], a["world"], a["port"], a["cfg"], a["pairs"], a["out"])
