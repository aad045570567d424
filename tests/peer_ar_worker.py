"""Worker for tests/test_peer_allreduce_gpu.py::test_tp_decode_peer_allreduce_two_ranks:
two ranks share cuda:0 (gloo for the host side, CUDA IPC for the peer regions)."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = BlockConfig(name="tp-test", n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, hidden=1024,
                      n_experts=8, n_shared=0, top_k=2, inter=1792)
    deg = PlanDegrees(world, 1, world, 1, 1)  # pure TP
    W = synthetic_weights(cfg, "cuda", seed=0)
    B, L = 16, 96
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = torch.randn(B, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    res = {}
    for peer in ("0", "1"):
        os.environ["HAP_PEER_AR"] = peer
        blk = HapMoEBlock(cfg, deg, None, rank=rank, weights=W)
        kv0, kv1 = blk.lay.kv_heads
        gk = torch.Generator(device="cuda")
        gk.manual_seed(4)
        kc = torch.randn(B, cfg.n_kv_heads, L, cfg.head_dim, device="cuda", generator=gk).to(torch.bfloat16)
        vc = torch.randn(B, cfg.n_kv_heads, L, cfg.head_dim, device="cuda", generator=gk).to(torch.bfloat16)
        cache = KVCache(kc[:, kv0:kv1].contiguous(), vc[:, kv0:kv1].contiguous())
        pos = torch.full((B,), L - 1, device="cuda", dtype=torch.int32)
        out = blk.forward(x.clone(), "decode", B, kv_cache=cache, positions=pos)
        torch.cuda.synchronize()
        res[peer] = out.float().cpu()
        if peer == "1":
            assert blk.graph_capturable(B)
            xs = x.clone()
            graph, gout = blk.capture_graph(xs, "decode", B, kv_cache=cache, positions=pos)
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize()
            res["graph"] = gout.float().cpu()
        blk.close()
        dist.barrier()
    err = float((res["1"] - res["0"]).abs().max() / res["0"].abs().max())
    ok = err < 2e-2 and torch.equal(res["1"], res["graph"])
    torch.save({"ok": ok, "err": err}, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    a = json.loads(sys.argv[1])
    main(a["rank"], a["world"], a["port"], a["out"])
