"""Worker for tests/test_ep_peer_gpu.py: several ranks share cuda:0 (gloo for the
host-side collectives, CUDA IPC for the peer-mapped buffers)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(rank, world, port, cfg_kw, plan, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.executor import HapMoEBlock
    from paper_2508_19373_b200.layout import PlanDegrees, replica_sequences
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = BlockConfig(**cfg_kw)
    deg = PlanDegrees(*plan)
    W = synthetic_weights(cfg, "cuda", seed=0)
    B, S = 4, 64
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    res = {}
    for peer in (False, True):
        blk = HapMoEBlock(cfg, deg, None, rank=rank, weights=W)
        blk.ep_peer = peer
        s0, s1 = replica_sequences(B, deg.a_dp, blk.lay.a_rep)
        outs = [blk.forward(x[s0 * S:s1 * S].contiguous(), "prefill", B, S) for _ in range(2)]
        torch.cuda.synchronize()
        res[peer] = [o.cpu() for o in outs]
        blk.close()
        dist.barrier()
    # the peer path must reproduce the all-to-all path exactly (same rows, same GEMMs), twice in a row
    ok = all(torch.equal(a, b) for a, b in zip(res[False], res[True])) and torch.equal(res[True][0], res[True][1])
    torch.save({"rank": rank, "ok": ok, "a_rep": blk.lay.a_rep, "out": res[True][0]}, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import json

    a = json.loads(sys.argv[1])
    main(a["rank"], a["world"], a["port"], a["cfg"], tuple(a["plan"]), a["out"])
