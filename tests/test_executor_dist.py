"""Multi-rank executor on CPU (gloo, world sizes 2 and 4): every plan in the
reference catalog gives the same block output as the single-device run.

The reference models these layouts only analytically (devices are integers,
transition.py:172); here the executor's actual collective schedule —
attention-TP AllReduce, DP->TP all-gather, EP count exchange + dispatch /
combine All-to-All, TP reduce-scatter and the final all-gather — runs on
real process groups.  Compute uses the test double tests/cpu_ops.py (the
sm_100a kernels cannot run here); the GPU path of the same executor is
covered by tests/test_block_gpu.py.
"""

import socket
from dataclasses import asdict

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import dist_worker
from cpu_ops import CpuOps

MIXTRAL_T = dict(name="mixtral-test", n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=64, hidden=256,
                 n_experts=8, n_shared=0, top_k=2, inter=256)
QWEN_T = dict(name="qwen-test", n_layers=2, n_q_heads=4, n_kv_heads=4, head_dim=64, hidden=256, n_experts=8,
              n_shared=2, top_k=4, inter=128, norm_topk_prob=False, qkv_bias=True, rms_eps=1e-6)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def catalog_plans(cfg, n):
    """Every (attention, expert) pair of the reference catalog (allow_expert_dp)."""
    from paper_2508_19373_b200.config import b200_hardware, import_moeplan

    mp_ = import_moeplan()
    cat = mp_.build_catalog(cfg.to_model_spec(), b200_hardware(n), allow_expert_dp=True)
    return [(a.tp_degree, a.dp_degree, e.tp_degree, e.ep_degree, e.dp_degree) for a in cat.attention
            for e in cat.expert]


def single_device(cfg):
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.weights import synthetic_weights

    W = synthetic_weights(cfg, "cpu", seed=0)
    blk, out, outd = dist_worker.run_plan(cfg, PlanDegrees(1, 1, 1, 1, 1), 0, W, CpuOps())
    return blk, out.float().numpy(), outd.float().numpy()


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("cfg_kw", [MIXTRAL_T, QWEN_T], ids=["mixtral", "qwen"])
@pytest.mark.parametrize("world", [2, 4])
def test_every_catalog_plan_matches_single_device(cfg_kw, world, tmp_path):
    from paper_2508_19373_b200.config import BlockConfig

    cfg = BlockConfig(**cfg_kw)
    plans = catalog_plans(cfg, world)
    assert len(plans) >= 4
    out_path = tmp_path / "res.npz"
    mp.spawn(dist_worker.worker, args=(world, free_port(), cfg_kw, plans, str(out_path)), nprocs=world, join=True)
    res = np.load(out_path)
    _, ref, refd = single_device(cfg)
    for p in plans:
        from paper_2508_19373_b200.layout import PlanDegrees

        lab = PlanDegrees(*p).label()
        got = res[lab]
        assert got.shape == ref.shape, lab
        # partial sums are reduced in bf16 across ranks: bf16-level tolerance
        assert rel(got, ref) < 3e-2, (lab, rel(got, ref))
        assert rel(res[lab + "|decode"], refd) < 3e-2, (lab, "decode")


def test_single_device_cpu_double_matches_oracle():
    """The CPU test double itself agrees with the numpy oracle (so the
    multi-rank comparisons above are anchored)."""
    from oracle import moe_block as O
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.weights import synthetic_weights

    from paper_2508_19373_b200.executor import HapMoEBlock
    from paper_2508_19373_b200.layout import PlanDegrees

    cfg = BlockConfig(**QWEN_T)
    Wt = synthetic_weights(cfg, "cpu", seed=0)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1, 1), None, device="cpu", weights=Wt, ops=CpuOps())
    x, *_ = dist_worker.make_inputs(cfg)
    out = blk.forward(x, "prefill", dist_worker.B, dist_worker.S).float().numpy()
    W = {k: v.float().numpy() for k, v in Wt.items()}
    spec = O.BlockSpec(hidden=cfg.hidden, n_q_heads=cfg.n_q_heads, n_kv_heads=cfg.n_kv_heads,
                       head_dim=cfg.head_dim, n_experts=cfg.n_experts, top_k=cfg.top_k, inter=cfg.inter,
                       n_shared=cfg.n_shared, norm_topk_prob=cfg.norm_topk_prob, qkv_bias=cfg.qkv_bias,
                       rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    x, *_ = dist_worker.make_inputs(cfg)
    ref = O.block_forward(spec, W, x.float().numpy(), dist_worker.B, bf16_mirror=True)
    idx = blk.last_routing[0].numpy()
    agree = (np.sort(ref["topk_idx"], 1) == np.sort(idx, 1)).all(1)
    assert agree.mean() >= 0.95
    assert rel(out[agree], ref["out"][agree]) < 2e-2
