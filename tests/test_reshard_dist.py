"""Prefill->decode expert layout switch (reshard) on gloo, world sizes 2 and 4.

For every ordered pair of expert strategies in the reference catalog, the
all-to-all reshard must reproduce the destination layout's weights exactly,
and the worst device's received bytes must equal the reference's
reshard_volume (transition.py:153-177) per layer.
"""

import json
import socket

import pytest
import torch.multiprocessing as mp

import dist_worker
from test_executor_dist import MIXTRAL_T, QWEN_T, free_port


@pytest.mark.parametrize("cfg_kw", [MIXTRAL_T, QWEN_T], ids=["mixtral", "qwen"])
@pytest.mark.parametrize("world", [2, 4])
def test_reshard_matches_direct_pack_and_reference_volume(cfg_kw, world, tmp_path):
    from paper_2508_19373_b200.config import BlockConfig, b200_hardware, import_moeplan

    mpl = import_moeplan()
    cfg = BlockConfig(**cfg_kw)
    cat = mpl.build_catalog(cfg.to_model_spec(), b200_hardware(world), allow_expert_dp=True)
    strat = [(e.tp_degree, e.ep_degree, e.dp_degree) for e in cat.expert]
    pairs = [(a, b) for a in strat for b in strat if a != b]
    out = tmp_path / "recv.json"
    mp.spawn(dist_worker.reshard_worker, args=(world, free_port(), cfg_kw, pairs, str(out)), nprocs=world, join=True)
    worst = json.loads(out.read_text())
    spec = cfg.to_model_spec()
    for a, b in pairs:
        src = mpl.ExpertStrategy(tp_degree=a[0], ep_degree=a[1], dp_degree=a[2])
        dst = mpl.ExpertStrategy(tp_degree=b[0], ep_degree=b[1], dp_degree=b[2])
        ref = mpl.reshard_volume(src, dst, spec)  # all layers
        key = f"{a[0]},{a[1]},{a[2]}->{b[0]},{b[1]},{b[2]}"
        assert worst[key] * spec.n_layers == ref, (key, worst[key], ref)


@pytest.mark.parametrize("prefill_deg,decode_deg", [((1, 2, 1, 2, 1), (1, 2, 2, 1, 1)),   # DP+EP -> DP+TP
                                                    ((2, 1, 2, 1, 1), (2, 1, 1, 2, 1))])  # TP+TP -> TP+EP
def test_model_stage_switch_matches_single_device(prefill_deg, decode_deg, tmp_path):
    """A stage-specific plan (prefill and decode expert layouts differ, the
    case planner.py:159-163 emits and tests/test_planner.py:330-351 pins):
    prefill, reshard, decode on 2 gloo ranks == the single-device model."""
    import numpy as np

    from cpu_ops import CpuOps
    from paper_2508_19373_b200.config import BlockConfig
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.model import HapModel

    out = tmp_path / "m.npz"
    mp.spawn(dist_worker.model_switch_worker, args=(2, free_port(), MIXTRAL_T, prefill_deg, decode_deg, str(out)),
             nprocs=2, join=True)
    got = np.load(out)
    cfg = BlockConfig(**MIXTRAL_T)
    ref_model = HapModel(cfg, PlanDegrees(1, 1, 1, 1, 1), None, n_layers=2, device="cpu", seed=3, ops=CpuOps())
    ref, refd = dist_worker.run_model(ref_model, cfg, 0, 1, None)

    def rel(a, b):
        return float(np.abs(a - b).max() / np.abs(b).max())

    assert rel(got["prefill"], ref) < 3e-2
    assert rel(got["decode"], refd) < 3e-2
