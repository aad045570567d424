"""Planner integration: the executor consumes moeplan's plan unchanged.

Pins the SURVEY.md §0/§8 observations on a B200 roofline profile: HAP picks
attention-DP + expert-TP for Mixtral 8x2048 at N >= 2; the pure-TP baseline
is the reference's baseline_indices(catalog, "tp"); Qwen2-57B at N = 8 has no
pure-TP attention; Qwen1.5 has no EP = 8; the forced DP -> EP plan of the
Mixtral-8x22B config exists in the catalog.
"""

import pytest

from paper_2508_19373_b200.config import PRESETS, b200_hardware, get_config, import_moeplan
from paper_2508_19373_b200.plan import baseline_plan, find_plan, plan_for, stage_plan

mp = import_moeplan()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_hap_picks_attention_dp_expert_tp_for_mixtral(n):
    res = plan_for(get_config("mixtral-8x7b"), n, 8, 2048, 0)
    sp = stage_plan(res, "prefill")
    assert (sp.attention.tp_degree, sp.attention.dp_degree) == (1, n)
    assert (sp.expert.tp_degree, sp.expert.ep_degree) == (n, 1)
    tp = baseline_plan(res, "tp")
    assert (tp.attention.tp_degree, tp.expert.tp_degree) == (n, n)
    # predicted HAP speedup over TP (reference simulate.compare, simulate.py:151-171);
    # 1.035 / 1.099 / 1.204x at N = 2 / 4 / 8 on the roofline profile
    rep = mp.compare([("hap", res.plan.indices()), ("tp", mp.baseline_indices(res.catalog, "tp"))], res.tensors,
                     get_config("mixtral-8x7b").to_model_spec(), mp.InferenceScenario(8, 2048, 0))
    assert rep.speedup("hap", "tp") > 1.0


def test_plan_result_drops_into_executor_types():
    from paper_2508_19373_b200.layout import PlanDegrees

    res = plan_for(get_config("mixtral-8x7b"), 8, 64, 1024, 2048)
    sp = stage_plan(res, "decode")
    deg = sp.degrees
    assert isinstance(deg, PlanDegrees) and deg.n == 8
    assert sp.expert is res.plan.expert_decode


def test_qwen2_57b_has_no_pure_tp_attention_at_8():
    res = plan_for(get_config("qwen2-57b-a14b"), 8, 64, 1024, 2048)
    with pytest.raises(mp.InfeasibleError):
        baseline_plan(res, "tp")
    assert max(a.tp_degree for a in res.catalog.attention) == 4


def test_qwen15_ep_catalog():
    res = plan_for(get_config("qwen1.5-moe-a2.7b"), 8, 8, 2048, 0)
    combos = {(e.tp_degree, e.ep_degree) for e in res.catalog.expert}
    assert combos == {(2, 4), (4, 2), (8, 1)}


def test_forced_dp_ep_plan_for_mixtral_8x22b():
    res = plan_for(get_config("mixtral-8x22b"), 8, 16, 4096, 0)
    forced = find_plan(res, attn_tp=1, exp_tp=1, exp_ep=8)
    assert forced is not None and forced.degrees.e_ep == 8 and forced.degrees.a_dp == 8


def test_all_presets_plan_on_b200():
    for name, cfg in PRESETS.items():
        for n in (1, 2, 4, 8):
            try:
                res = plan_for(cfg, n, 8, 512, 64)
            except mp.InfeasibleError:
                continue
            assert res.plan.predicted_total_s > 0


def test_b200_profile():
    hw = b200_hardware(8)
    assert hw.n_devices == 8 and hw.peak_flops == pytest.approx(1.6525e15)
    assert hw.link_label == "nvlink5"
