"""Expert reshard phases without a process group (CPU): every rank's
reshard_pack is routed to its receivers by hand (what all_to_all_single does)
and reshard_unpack must reproduce the destination layout's packed weights
exactly — for the direct-copy fast path (slices on whole SwiGLU blocks) and
the generic path alike, at N = 2, 4, 8."""

import pytest
import torch

from paper_2508_19373_b200.config import BlockConfig
from paper_2508_19373_b200.layout import PlanDegrees, RankLayout
from paper_2508_19373_b200.transition import reshard_pack, reshard_unpack
from paper_2508_19373_b200.weights import pack_rank_weights, synthetic_weights

FAST = dict(name="rs-fast", n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=64, hidden=128, n_experts=8,
            n_shared=0, top_k=2, inter=2048)
SHARED = dict(name="rs-shared", n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=64, hidden=128, n_experts=8,
              n_shared=2, top_k=4, inter=1024, norm_topk_prob=False, qkv_bias=True)
GENERIC = dict(name="rs-generic", n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=64, hidden=128, n_experts=8,
               n_shared=1, top_k=2, inter=352)


def _simulate(cfg, n, src, dst, device="cpu"):
    W = synthetic_weights(cfg, device, seed=0)
    lay = lambda te, r: RankLayout(PlanDegrees(1, n, te[0], te[1], 1), r, cfg.n_q_heads, cfg.n_kv_heads,  # noqa: E731
                                   cfg.n_experts, cfg.inter, cfg.n_shared)
    packs = [reshard_pack(cfg, pack_rank_weights(cfg, W, lay(src, r)), lay(src, r), lay(dst, r)) for r in range(n)]
    for r in range(n):
        # the all-to-all: rank r receives, in source order, the chunk each source addressed to it
        chunks = []
        for q in range(n):
            send, ins, _, _ = packs[q]
            off = sum(ins[:r])
            chunks.append(send[off:off + ins[r]])
        got = reshard_unpack(packs[r][3], torch.cat(chunks))
        want = pack_rank_weights(cfg, W, lay(dst, r))
        for name in ("w13", "w2", "ws13", "ws2"):
            a, b = getattr(got, name), getattr(want, name)
            assert (a is None) == (b is None), name
            if a is not None:
                assert a.shape == b.shape and torch.equal(a, b), (cfg.name, n, src, dst, r, name)
        assert got.hw == want.hw and got.hw_s == want.hw_s and got.inter_local == want.inter_local


@pytest.mark.parametrize("cfg_kw", [FAST, SHARED, GENERIC], ids=["fast", "shared", "generic"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_reshard_phases_reproduce_destination_layout(cfg_kw, n):
    cfg = BlockConfig(**cfg_kw)
    # expert-TP degrees whose slice admits a SwiGLU tile width (a multiple of 8)
    strat = [(t, n // t) for t in (1, 2, 4, 8) if t <= n and n % t == 0 and (cfg.inter // t) % 8 == 0]
    for src in strat:
        for dst in strat:
            if src != dst:
                _simulate(cfg, n, src, dst)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_kw", [FAST, SHARED, GENERIC], ids=["fast", "shared", "generic"])
def test_reshard_phases_on_gpu(cfg_kw):
    """The same phases with the weights on the GPU: pack and unpack run as
    batched hap_copy2d_batched launches (bit-identical weights); the second
    pass over fresh weight tensors replays the compiled copy records (the
    per-layer path of a stage switch) and must be bit-identical too."""
    from paper_2508_19373_b200 import ops, transition

    cfg = BlockConfig(**cfg_kw)
    transition._COPY_PLANS.clear()
    before = ops.LAUNCHES[0]
    for rep in range(2):
        for n in (2, 8):
            strat = [(t, n // t) for t in (1, 2, 4, 8) if t <= n and n % t == 0 and (cfg.inter // t) % 8 == 0]
            for src in strat:
                for dst in strat:
                    if src != dst:
                        _simulate(cfg, n, src, dst, device="cuda")
        if rep == 0:
            n_plans = len(transition._COPY_PLANS)
    assert ops.LAUNCHES[0] > before
    assert len(transition._COPY_PLANS) == n_plans  # the second pass compiled nothing new
    if cfg.name != "rs-generic":
        assert n_plans > 0


def test_rows_split_views():
    """The descriptor rule of ops.copy_views: uniform-pitch stacks of
    contiguous rows are found (merging trailing dims), anything else is None."""
    from paper_2508_19373_b200.ops import _rows_split

    t = torch.empty(8, 2, 4, 16)
    v = t[:, 0]                              # [8, 4, 16] blocks, pitch 2*4*16
    c = torch.empty(8, 4, 16)
    assert _rows_split(v.shape, v.stride(), c.stride()) == (8, 64, 128, 64)
    assert _rows_split(c.shape, c.stride(), c.stride()) == (1, 512, 512, 512)
    w = torch.empty(32, 100)[:, 10:30]       # column block of a row-major matrix
    d = torch.empty(32, 20)
    assert _rows_split(w.shape, w.stride(), d.stride()) == (32, 20, 100, 20)
    assert _rows_split(w.t().shape, w.t().stride(), d.t().contiguous().stride()) is None
