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


def reshard_worker(rank, world, port, cfg_kwargs, pairs, out_path):
    """For every (src, dst) expert layout pair: reshard_expert_weights must equal
    packing the destination layout directly; record received bytes per rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.layout import PlanDegrees, RankLayout
    from paper_2508_19373_b200.transition import reshard_expert_weights
    from paper_2508_19373_b200.weights import pack_rank_weights, synthetic_weights

    cfg = BlockConfig(**cfg_kwargs)
    W = synthetic_weights(cfg, "cpu", seed=0)
    recv = {}
    for (ti, ei, di), (tj, ej, dj) in pairs:
        mk = lambda t, e, d: RankLayout(PlanDegrees(1, world, t, e, d), rank, cfg.n_q_heads, cfg.n_kv_heads,  # noqa: E731
                                        cfg.n_experts, cfg.inter, cfg.n_shared)
        li, lj = mk(ti, ei, di), mk(tj, ej, dj)
        wi = pack_rank_weights(cfg, W, li)
        got = reshard_expert_weights(cfg, wi, li, lj)
        want = pack_rank_weights(cfg, W, lj)
        for name in ("w13", "w2", "ws13", "ws2"):
            a, b = getattr(got, name), getattr(want, name)
            assert (a is None) == (b is None), name
            if a is not None:
                assert a.shape == b.shape and torch.equal(a, b), (name, (ti, ei, di), (tj, ej, dj))
        assert got.hw == want.hw and got.inter_local == want.inter_local
        # bytes this rank received (one layer)
        from math import gcd
        from paper_2508_19373_b200.transition import _owned
        ns = ti * tj // gcd(ti, tj)
        missing = len(_owned(lj, ns) - _owned(li, ns))
        recv[f"{ti},{ei},{di}->{tj},{ej},{dj}"] = missing * 3 * (cfg.inter // ns) * cfg.hidden * 2
    objs = [None] * world
    dist.all_gather_object(objs, recv)
    if rank == 0:
        import json
        worst = {k: max(o[k] for o in objs) for k in objs[0]}
        Path(out_path).write_text(json.dumps(worst))
    dist.barrier()
    dist.destroy_process_group()


def model_switch_worker(rank, world, port, cfg_kwargs, prefill_deg, decode_deg, out_path):
    """2-layer model: prefill under one expert layout, reshard (stage switch),
    decode under another; rank 0 saves the assembled outputs."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    from cpu_ops import CpuOps
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.layout import PlanDegrees, replica_sequences
    from paper_2508_19373_b200.model import HapModel

    class _E:  # strategy-like object for switch_expert_layout
        def __init__(self, t, e, d):
            self.tp_degree, self.ep_degree, self.dp_degree = t, e, d

    cfg = BlockConfig(**cfg_kwargs)
    model = HapModel(cfg, PlanDegrees(*prefill_deg), None, n_layers=2, rank=rank, device="cpu", seed=3, ops=CpuOps())
    out, outd = run_model(model, cfg, rank, world, _E(*decode_deg[2:]))
    if rank == 0:
        np.savez(out_path, prefill=out, decode=outd)
    dist.barrier()
    dist.destroy_process_group()


def run_model(model, cfg, rank, world, decode_expert):
    from paper_2508_19373_b200.layout import replica_sequences

    x, xd, _, _ = make_inputs(cfg)
    deg = model.deg
    s0, s1 = replica_sequences(B, deg.a_dp, model.lay.a_rep)
    caches = model.new_caches(B, S + 4)
    out = model.prefill(x[s0 * S:s1 * S].contiguous(), B, S, caches)
    if decode_expert is not None:
        model.switch_expert_layout(decode_expert)
    pos = torch.full((s1 - s0,), S, dtype=torch.int32)
    outd = model.decode_step(xd[s0:s1].contiguous(), B, caches, pos)
    if world > 1:
        objs = [None] * world
        dist.all_gather_object(objs, (model.lay.a_rep, out.float().numpy(), outd.float().numpy()))
        reps = {}
        for a, o, od in objs:
            reps.setdefault(a, (o, od))
        keys = sorted(reps)
        return np.concatenate([reps[k][0] for k in keys]), np.concatenate([reps[k][1] for k in keys])
    return out.float().numpy(), outd.float().numpy()
