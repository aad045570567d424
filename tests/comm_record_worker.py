"""Worker for tests/test_comm_schedule.py: runs every catalog plan (prefill and
decode) on gloo with the executor's collectives recorded as
(stage, kind, group, logical bytes) per rank."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def _recording(comm, log, stage):
    """Wrap a Comm so every collective call appends (stage, kind, group, bytes)."""
    def grp(kind):
        return list(comm.groups[kind][0])

    orig = {n: getattr(comm, n) for n in ("all_reduce", "all_gather", "reduce_scatter", "all_to_all")}

    def all_reduce(t, kind):
        if comm.size(kind) > 1:
            log.append((stage[0], "allreduce", grp(kind), t.numel() * t.element_size()))
        return orig["all_reduce"](t, kind)

    def all_gather(out, inp, kind):
        if comm.size(kind) > 1:
            log.append((stage[0], "allgather", grp(kind), out.numel() * out.element_size()))
        return orig["all_gather"](out, inp, kind)

    def reduce_scatter(out, inp, kind):
        if comm.size(kind) > 1:
            log.append((stage[0], "reduce_scatter", grp(kind), inp.numel() * inp.element_size()))
        return orig["reduce_scatter"](out, inp, kind)

    def all_to_all(out, inp, out_splits, in_splits, kind):
        if comm.size(kind) > 1:
            what = "count_exchange" if inp.dtype == torch.int32 else "all_to_all"
            log.append((stage[0], what, grp(kind), inp.numel() * inp.element_size()))
        return orig["all_to_all"](out, inp, out_splits, in_splits, kind)

    comm.all_reduce, comm.all_gather = all_reduce, all_gather
    comm.reduce_scatter, comm.all_to_all = reduce_scatter, all_to_all


def worker(rank, world, port, cfg_kwargs, plans, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    import dist_worker
    from cpu_ops import CpuOps
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.executor import HapMoEBlock, KVCache
    from paper_2508_19373_b200.layout import PlanDegrees, replica_sequences
    from paper_2508_19373_b200.weights import synthetic_weights

    cfg = BlockConfig(**cfg_kwargs)
    W = synthetic_weights(cfg, "cpu", seed=0)
    x, xd, kc, vc = dist_worker.make_inputs(cfg)
    B, S, DB = dist_worker.B, dist_worker.S, dist_worker.DEC_B
    res = {}
    for p in plans:
        deg = PlanDegrees(*p)
        blk = HapMoEBlock(cfg, deg, None, rank=rank, device="cpu", weights=W, ops=CpuOps())
        log, stage = [], ["prefill"]
        _recording(blk.comm, log, stage)
        s0, s1 = replica_sequences(B, deg.a_dp, blk.lay.a_rep)
        blk.forward(x[s0 * S:s1 * S].contiguous(), "prefill", B, S)
        stage[0] = "decode"
        d0, d1 = replica_sequences(DB, deg.a_dp, blk.lay.a_rep)
        k0, k1 = blk.lay.kv_heads
        cache = KVCache(kc[d0:d1, k0:k1].contiguous(), vc[d0:d1, k0:k1].contiguous())
        pos = torch.tensor(dist_worker.DEC_POS[d0:d1], dtype=torch.int32)
        blk.forward(xd[d0:d1].contiguous(), "decode", DB, kv_cache=cache, positions=pos)
        objs = [None] * world
        dist.all_gather_object(objs, log)
        res[json.dumps(list(p))] = objs
    if rank == 0:
        Path(out_path).write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()
