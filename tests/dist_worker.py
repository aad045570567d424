"""Worker for the gloo multi-process executor tests (spawned by test_executor_dist.py)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

B, S = 4, 16
DEC_B, DEC_L = 4, 24
DEC_POS = [3, 9, 17, 23]


def make_inputs(cfg):
    g = torch.Generator().manual_seed(1)
    x = torch.randn(B * S, cfg.hidden, generator=g).to(torch.bfloat16)
    xd = torch.randn(DEC_B, cfg.hidden, generator=g).to(torch.bfloat16)
    kc = torch.randn(DEC_B, cfg.n_kv_heads, DEC_L, cfg.head_dim, generator=g).to(torch.bfloat16)
    vc = torch.randn(DEC_B, cfg.n_kv_heads, DEC_L, cfg.head_dim, generator=g).to(torch.bfloat16)
    return x, xd, kc, vc


def run_plan(cfg, deg, rank, W, ops):
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import replica_sequences

    x, xd, kc, vc = make_inputs(cfg)
    blk = HapMoEBlock(cfg, deg, None, rank=rank, device="cpu", weights=W, ops=ops)
    s0, s1 = replica_sequences(B, deg.a_dp, blk.lay.a_rep)
    out = blk.forward(x[s0 * S:s1 * S].contiguous(), "prefill", B, S)
    d0, d1 = replica_sequences(DEC_B, deg.a_dp, blk.lay.a_rep)
    k0, k1 = blk.lay.kv_heads
    cache = KVCache(kc[d0:d1, k0:k1].contiguous(), vc[d0:d1, k0:k1].contiguous())
    pos = torch.tensor(DEC_POS[d0:d1], dtype=torch.int32)
    outd = blk.forward(xd[d0:d1].contiguous(), "decode", DEC_B, kv_cache=cache, positions=pos)
    return blk, out, outd


def assemble(world, blk, out, outd):
    objs = [None] * world
    dist.all_gather_object(objs, (blk.lay.a_rep, blk.lay.a_tp_rank, out.float().numpy(), outd.float().numpy()))
    reps = {}
    for a_rep, tpr, o, od in objs:
        if a_rep in reps:
            # every rank of an attention replica must hold the identical block output
            assert np.array_equal(reps[a_rep][0], o) and np.array_equal(reps[a_rep][1], od)
        else:
            reps[a_rep] = (o, od)
    keys = sorted(reps)
    return np.concatenate([reps[k][0] for k in keys]), np.concatenate([reps[k][1] for k in keys])


def worker(rank, world, port, cfg_kwargs, plans, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    from cpu_ops import CpuOps
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = BlockConfig(**cfg_kwargs)
    W = synthetic_weights(cfg, "cpu", seed=0)
    res = {}
    for p in plans:
        deg = PlanDegrees(*p)
        blk, out, outd = run_plan(cfg, deg, rank, W, CpuOps())
        full, fulld = assemble(world, blk, out, outd)
        res[deg.label()] = full
        res[deg.label() + "|decode"] = fulld
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()
