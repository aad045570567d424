"""Planner integration: the reference ILP (moeplan) picks the plan the executor runs.

``plan_for`` is ``moeplan.plan`` (planner.py:527-549) on a B200
HardwareProfile; ``baseline_plan`` builds the reference's pure-TP comparison
plan from ``baseline_indices`` (planner.py:486-517).  Both return moeplan
objects unchanged, so any Plan from solve_ilp / solve_bruteforce drops into
``HapMoEBlock.from_plan``.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Optional

from .config import BlockConfig, b200_hardware, import_moeplan
from .layout import PlanDegrees


@dataclass(frozen=True)
class StagePlan:
    attention: object   # moeplan AttentionStrategy
    expert: object      # moeplan ExpertStrategy

    @property
    def degrees(self) -> PlanDegrees:
        return PlanDegrees.from_strategies(self.attention, self.expert)

    def label(self) -> str:
        return f"{self.attention.label()}+{self.expert.label()}"


def plan_for(cfg: BlockConfig, n_devices: int, batch: int, input_len: int, output_len: int = 0,
             cost_models=None, hw=None, **opts):
    """moeplan.plan() for this block on n_devices B200s; returns PlanResult."""
    mp = import_moeplan()
    hw = hw or b200_hardware(n_devices)
    scen = mp.InferenceScenario(batch=batch, input_len=input_len, output_len=output_len)
    po = mp.PlanOptions(cost_models=cost_models or mp.CostModels(), **opts)
    return mp.plan(cfg.to_model_spec(), hw, scen, po)


def stage_plan(result, stage: str) -> StagePlan:
    p = result.plan
    return StagePlan(p.attention, p.expert_prefill if stage == "prefill" else p.expert_decode)


def baseline_plan(result, name: str = "tp", stage: str = "prefill") -> StagePlan:
    """The reference's named comparison plan (tp / ep / dp) inside the same catalog."""
    mp = import_moeplan()
    k, i, j = mp.baseline_indices(result.catalog, name)
    cat = result.catalog
    return StagePlan(cat.attention[k], cat.expert[i if stage == "prefill" else j])


CALIBRATION_FILE = Path(__file__).resolve().parent.parent / "profiles" / "r02_calibration.json"


def calibrated_plan(cfg: BlockConfig, n_devices: int, batch: int, input_len: int, output_len: int = 0,
                    path: Optional[Path] = None, hw=None, routing: str = "balanced"):
    """The reference ILP re-solved on B200-measured module tables
    (calib.measured_cost_tensors): returns (PlanResult-like, source) where
    source says whether measured tables were found for this exact scenario.
    routing: which measured expert cells ("balanced" = the synthetic workload
    the bench runs, "skewed" = the imbalanced-routing workload)."""
    import json

    from . import calib

    mp = import_moeplan()
    res = plan_for(cfg, n_devices, batch, input_len, output_len, hw=hw)
    p = Path(path) if path else CALIBRATION_FILE
    if not p.exists():
        return res, "roofline (no calibration file)"
    doc = json.loads(p.read_text())
    case = next((c for c in doc.get("cases", []) if c.get("model") == cfg.name and c.get("n") == n_devices
                 and c.get("scenario") == {"batch": batch, "input_len": input_len, "output_len": output_len}
                 and c.get("routing", "balanced") == routing and "cells" in c), None)
    if case is None:
        return res, "roofline (scenario not calibrated)"
    att = {a.label(): k for k, a in enumerate(res.catalog.attention)}
    exp = {e.label(): i for i, e in enumerate(res.catalog.expert)}
    meas = []
    for cell in case["cells"]:
        idx = att.get(cell["strategy"]) if cell["module"] == "attention" else exp.get(cell["strategy"])
        if idx is None:
            continue
        meas.append(calib.Measurement(cfg.name, n_devices, cell["module"], cell["stage"], cell["strategy"], idx,
                                      0, 0, 0, 0, cell["measured_us"] * 1e-6, cell["roofline_us"] * 1e-6))
    tens = calib.measured_cost_tensors(res, meas)
    scen = mp.InferenceScenario(batch=batch, input_len=input_len, output_len=output_len)
    sel = mp.solve_ilp(tens, scen, cfg.to_model_spec(), res.catalog)
    return mp.PlanResult(plan=sel, tensors=tens, catalog=res.catalog), f"measured B200 tables ({p.name}, {routing})"


def find_plan(result, attn_tp: int, exp_tp: int, exp_ep: int, exp_dp: int = 1) -> Optional[StagePlan]:
    """A specific catalog entry (e.g. the forced DP->EP plan of the Mixtral-8x22B config)."""
    cat = result.catalog
    a = next((s for s in cat.attention if s.tp_degree == attn_tp), None)
    e = next((s for s in cat.expert if (s.tp_degree, s.ep_degree, s.dp_degree) == (exp_tp, exp_ep, exp_dp)), None)
    return StagePlan(a, e) if a is not None and e is not None else None
