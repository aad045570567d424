"""Collective-schedule conformance: the collectives the executor actually issues
for every catalog plan match the reference's per-layer charge
``comm_volume`` (strategies.py:296-344) and its ``wire_bytes`` model
(strategies.py:274-285).

Recorded on gloo (world 2 and 4, every catalog plan incl. expert-DP, prefill
and decode) through tests/comm_record_worker.py.  The executor realises the
reference's rows as follows:

* attention AllReduce (w / a_dp over the attention-TP group) — issued as an
  AllReduce, or, when the expert tp is 1 (EP or expert-DP shards of 1/a_tp of
  the replica), as a ReduceScatter straight onto the shards plus the
  AllGather after the experts (the same wire bytes);
* EP dispatch + combine All-to-All (k * w_exp each over the EP group) —
  issued exactly (logical volume = the EP group's summed inputs), plus the
  count exchange (E int32 per rank, not modelled by the reference);
* DP->TP boundary (two AllGathers of w over N) and the expert-TP AllReduce —
  issued as an AllGather over the gather group, a ReduceScatter over the
  expert-TP group and an AllGather over the attention-TP group.  The per-device
  wire bytes (all reductions and gathers together) equal the reference's for
  every plan with expert tp 1 or without EP / expert DP (pure TP; attention
  DP/hybrid x expert TP), and never exceed them otherwise:
  under EP x TP each TP group reduces only its own shard (w / ep), where the
  reference charges an AllReduce of the whole w.

Row padding: a replica's rows are padded to a multiple of N
(layout.tokens_per_replica), so bytes are compared against the reference's
w scaled by the padded/real token ratio.
"""

import json
import socket

import pytest
import torch.multiprocessing as mp

import comm_record_worker
from test_executor_dist import MIXTRAL_T, catalog_plans


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _wire(kind, nbytes, g):
    if g <= 1:
        return 0.0
    if kind == "allreduce":
        return 2.0 * nbytes * (g - 1) / g
    if kind in ("allgather", "reduce_scatter"):
        return nbytes * (g - 1) / g
    raise ValueError(kind)


@pytest.mark.parametrize("world", [2, 4])
def test_issued_collectives_match_comm_volume(world, tmp_path):
    from paper_2508_19373_b200.config import BlockConfig, b200_hardware, import_moeplan
    from paper_2508_19373_b200.layout import PlanDegrees, tokens_per_replica

    import dist_worker

    mp_ = import_moeplan()
    cfg = BlockConfig(**MIXTRAL_T)
    spec = cfg.to_model_spec()
    cat = mp_.build_catalog(spec, b200_hardware(world), allow_expert_dp=True)
    plans = catalog_plans(cfg, world)
    out = tmp_path / "log.json"
    mp.spawn(comm_record_worker.worker, args=(world, free_port(), MIXTRAL_T, plans, str(out)), nprocs=world,
             join=True)
    logs = json.loads(out.read_text())
    stages = {"prefill": (dist_worker.B, dist_worker.S), "decode": (dist_worker.DEC_B, 1)}
    checked = 0
    for p in plans:
        deg = PlanDegrees(*p)
        attn = next(a for a in cat.attention if (a.tp_degree, a.dp_degree) == (deg.a_tp, deg.a_dp))
        exp = next(e for e in cat.expert if (e.tp_degree, e.ep_degree, e.dp_degree) == (deg.e_tp, deg.e_ep, deg.e_dp))
        per_rank = logs[json.dumps(list(p))]
        for stage, (batch, seq) in stages.items():
            scen = mp_.InferenceScenario(batch=batch, input_len=seq if stage == "prefill" else 16,
                                         output_len=0 if stage == "prefill" else 8)
            ref = mp_.comm_volume(attn, exp, spec, scen, stage)
            T = batch * seq
            _, rows = tokens_per_replica(batch, deg.a_dp, seq, world)
            pad = rows * deg.a_dp / T
            ref_attn = [c for c in ref.collectives if c.side == "attention"]
            ref_a2a = [c for c in ref.collectives if c.kind == mp_.strategies.ALL_TO_ALL]
            ref_rest = sum(mp_.strategies.wire_bytes(c) for c in ref.collectives
                           if c.side != "attention" and c.kind != mp_.strategies.ALL_TO_ALL)
            a2a_inputs = {}
            for r, log in enumerate(per_rank):
                recs = [tuple(x) for x in log if x[0] == stage]
                kinds = {x[1] for x in recs}
                assert kinds <= {"allreduce", "allgather", "reduce_scatter", "all_to_all", "count_exchange"}, kinds
                # (1) attention AllReduce of w / a_dp over the attention-TP group: issued as an
                # all-reduce, or (expert tp 1) as a reduce-scatter onto the expert shards
                # whose AllGather back closes the same AllReduce
                first = [x for x in recs if x[1] in ("allreduce", "reduce_scatter")][:1]
                if deg.a_tp > 1:
                    assert len(ref_attn) == 1 and first, (deg.label(), stage)
                    _, kind, g, nb = first[0]
                    assert kind == ("reduce_scatter" if deg.e_tp == 1 else "allreduce"), (deg.label(), kind)
                    assert len(g) == ref_attn[0].group_size == deg.a_tp
                    assert nb == pytest.approx(ref_attn[0].tensor_bytes * pad), (deg.label(), stage)
                else:
                    assert not ref_attn, (deg.label(), stage)
                # (2) EP dispatch + combine
                a2a = [x for x in recs if x[1] == "all_to_all"]
                assert len(a2a) == len(ref_a2a) == (2 if deg.e_ep > 1 else 0), (deg.label(), stage)
                for i, (_, _, g, nb) in enumerate(a2a):
                    assert len(g) == deg.e_ep
                    a2a_inputs.setdefault((i, tuple(g)), []).append(nb)
                cnt = [x for x in recs if x[1] == "count_exchange"]
                assert len(cnt) == (1 if deg.e_ep > 1 else 0)
                # (3) every reduction / gather, per-device wire bytes, against the
                # reference's attention + boundary + expert-TP rows
                wire = sum(_wire(k, nb, len(g)) for _, k, g, nb in recs if k in ("allreduce", "allgather",
                                                                               "reduce_scatter"))
                ref_wire = ref_rest + sum(mp_.strategies.wire_bytes(c) for c in ref_attn)
                if deg.e_tp == 1 or (deg.e_ep == 1 and deg.e_dp == 1):
                    assert wire == pytest.approx(ref_wire * pad), (deg.label(), stage, wire, ref_wire)
                else:
                    assert wire <= ref_wire * pad + 1e-6, (deg.label(), stage, wire, ref_wire)
            for (i, g), nbs in a2a_inputs.items():
                assert len(nbs) == len(g)
                assert sum(nbs) == pytest.approx(ref_a2a[i].tensor_bytes * pad), (deg.label(), stage, i)
            checked += 1
    assert checked == 2 * len(plans)
