"""Worker for tests/test_boundary_peer_gpu.py: ranks share cuda:0 (gloo for the
host collectives of the reference path, CUDA IPC for the peer buffers)."""

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
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import PlanDegrees, replica_sequences
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = BlockConfig(**cfg_kw)
    deg = PlanDegrees(*plan)
    W = synthetic_weights(cfg, "cuda", seed=0)
    B, S, L = 4, 64, 96
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    xd = torch.randn(B, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    res = {}
    for peer in (False, True):
        blk = HapMoEBlock(cfg, deg, None, rank=rank, weights=W)
        blk.boundary_peer = peer
        assert blk._uses_peer_boundary() == peer
        s0, s1 = replica_sequences(B, deg.a_dp, blk.lay.a_rep)
        cache = KVCache.empty(s1 - s0, blk.w.n_kv_local, L, cfg.head_dim, "cuda")
        outs = [blk.forward(x[s0 * S:s1 * S].contiguous(), "prefill", B, S, kv_cache=cache) for _ in range(2)]
        pos = torch.full((s1 - s0,), S, device="cuda", dtype=torch.int32)
        xl = xd[s0:s1].contiguous()
        outd = blk.forward(xl, "decode", B, kv_cache=cache, positions=pos)
        torch.cuda.synchronize()
        res[peer] = {"prefill": [o.cpu() for o in outs], "decode": outd.cpu()}
        if peer:
            # no NCCL and no host sync on the peer boundary: the decode step captures into a CUDA graph
            assert blk.graph_capturable()
            graph, out_static = blk.capture_graph(xl, "decode", B, kv_cache=cache, positions=pos)
            reps = []
            for _ in range(2):
                graph.replay()
                torch.cuda.synchronize()
                reps.append(out_static.cpu())
            res[peer]["graph"] = reps
        blk.close()
        dist.barrier()
    a, b = res[False], res[True]
    rel = lambda u, v: float((u.float() - v.float()).abs().max() / v.float().abs().max())  # noqa: E731
    stats = {
        "prefill_rel": rel(b["prefill"][0], a["prefill"][0]),
        "decode_rel": rel(b["decode"], a["decode"]),
        "prefill_repeat_equal": torch.equal(b["prefill"][0], b["prefill"][1]),
        "graph_equal_eager": all(torch.equal(r, b["decode"]) for r in b["graph"]),
    }
    torch.save({"rank": rank, "stats": stats, "a_rep": blk.lay.a_rep, "out": b["prefill"][0]}, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import json

    a = json.loads(sys.argv[1])
    main(a["rank"], a["world"], a["port"], a["cfg"], tuple(a["plan"]), a["out"])
