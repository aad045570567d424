"""The executor's weight placement and rank groups follow the reference's
ownership contract (transition.py:127-150 ``_ownership``) for every catalog
entry of every BASELINE model at N = 1..8, and its token layouts are
consistent (every rank's expert shard is covered by its gather group or lies
inside its own attention replica)."""

import pytest

from paper_2508_19373_b200.config import PRESETS, b200_hardware, import_moeplan
from paper_2508_19373_b200.layout import PlanDegrees, RankLayout, tokens_per_replica

mp = import_moeplan()
from moeplan.transition import _ownership  # noqa: E402  (reference internal, the layout contract)


def catalog(cfg, n):
    try:
        return mp.build_catalog(cfg.to_model_spec(), b200_hardware(n), allow_expert_dp=True)
    except mp.InfeasibleError:
        return None


CASES = [(name, n) for name in sorted(PRESETS) for n in range(1, 9)]


@pytest.mark.parametrize("name,n", CASES)
def test_expert_ownership_matches_reference(name, n):
    cfg = PRESETS[name]
    cat = catalog(cfg, n)
    if cat is None:
        pytest.skip("no feasible catalog")
    for a in cat.attention:
        for e in cat.expert:
            deg = PlanDegrees.from_strategies(a, e)
            n_slices = e.tp_degree
            for r in range(n):
                lay = RankLayout(deg, r, cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.inter, cfg.n_shared)
                ref = _ownership(e, r, cfg.n_experts, cfg.n_shared, n_slices)
                e0, e1 = lay.experts
                i0, i1 = lay.inter_slice
                span = cfg.inter // n_slices
                mine = {(x, i0 // span) for x in range(e0, e1)}
                mine |= {(cfg.n_experts + u, i0 // span) for u in range(cfg.n_shared)}
                assert mine == ref, (name, n, deg.label(), r)
                assert (i1 - i0) == span
                # shared rows: per unit the same TP slice
                for u, (s0, s1) in enumerate(lay.shared_rows()):
                    assert (s0, s1) == (u * cfg.inter + i0, u * cfg.inter + i1)


@pytest.mark.parametrize("name,n", CASES)
def test_groups_partition_and_token_layout(name, n):
    cfg = PRESETS[name]
    cat = catalog(cfg, n)
    if cat is None:
        pytest.skip("no feasible catalog")
    for a in cat.attention:
        for e in cat.expert:
            deg = PlanDegrees.from_strategies(a, e)
            lays = [RankLayout(deg, r, cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.inter, cfg.n_shared)
                    for r in range(n)]
            for kind in ("attn_tp_group", "exp_tp_group", "gather_group", "a2a_group"):
                groups = lays[0].all_groups(kind)
                flat = sorted(r for g in groups for r in g)
                assert flat == list(range(n)), (kind, deg.label())
                for lay in lays:
                    assert lay.rank in getattr(lay, kind)()
            # attention heads: every q/kv head held by exactly dp ranks
            for lay in lays:
                q0, q1 = lay.q_heads
                assert (q1 - q0) * deg.a_tp == cfg.n_q_heads
            # expert shard coverage: S_e >= a_dp => shard inside own replica; else gather group spans
            _, rows = tokens_per_replica(8, deg.a_dp, 16, n)
            for lay in lays:
                S_e = lay.n_shards
                if S_e >= deg.a_dp:
                    assert lay.gather_group() == [lay.rank]
                    assert (S_e // deg.a_dp) * (rows // (S_e // deg.a_dp)) == rows
                else:
                    reps = sorted(lays[r].a_rep for r in lay.gather_group())
                    assert len(reps) == deg.a_dp // S_e and len(set(reps)) == len(reps)
                    assert lay.a_rep in reps
                # after the reduce-scatter each rank owns rows/a_tp rows of its replica
                assert rows % deg.a_tp == 0
            # EP groups: each a2a group holds every expert block exactly once
            if deg.e_ep > 1:
                for lay in lays:
                    blocks = sorted(lays[r].experts for r in lay.a2a_group())
                    assert blocks[0][0] == 0 and blocks[-1][1] == cfg.n_experts
                    assert all(blocks[i][1] == blocks[i + 1][0] for i in range(len(blocks) - 1))


def test_layout_rejects_invalid_plans():
    with pytest.raises(ValueError):
        RankLayout(PlanDegrees(3, 1, 3, 1), 0, 32, 8, 8, 14336, 0)  # tp not a power of two
    with pytest.raises(ValueError):
        RankLayout(PlanDegrees(8, 1, 1, 8), 0, 28, 4, 64, 2560, 8)   # tp 8 > 4 kv heads
    with pytest.raises(ValueError):
        RankLayout(PlanDegrees(1, 8, 1, 8), 0, 16, 16, 60, 1408, 4)  # ep 8 does not divide 60
    with pytest.raises(ValueError):
        RankLayout(PlanDegrees(1, 4, 1, 2, 2), 0, 32, 8, 8, 14336, 0)  # DP x EP
