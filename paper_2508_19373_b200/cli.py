"""Command line: plan / measure / run, in the reference CLI's conventions.

``python -m paper_2508_19373_b200 <command>`` mirrors ``moeplan``'s CLI
(reference cli.py): every run prints one JSON payload carrying a manifest
(resolved inputs, flags, tool version, wall time; cli.py:210-231), and exit
codes are the reference's — 0 success, 2 config error, 3 infeasible,
4 internal invariant breach (cli.py:55-58).

  plan     the reference ILP (moeplan.plan, planner.py:527-549) for a model on
           N B200s — hardware from ``presets/b200.cfg`` (the reference's
           ``[hardware]`` config format, configio.py:100-124) or ``--hw``;
           ``--calibrated`` re-solves on the B200-measured module tables.
  measure  times every (strategy, stage) cell the planner prices on this GPU
           with the product kernels and writes the reference's calibration
           CSV (``kind,b,s,h,volume,context,latency_s``, costmodel.py:307-332)
           — the input of ``moeplan calibrate`` / ``train_forest``.
  run      builds the block for the chosen plan on this GPU and times the
           prefill and decode forward (tokens/s), N = 1.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path
from typing import Dict, Optional

from .config import BlockConfig, get_config, import_moeplan

EXIT_OK, EXIT_CONFIG, EXIT_INFEASIBLE, EXIT_INTERNAL = 0, 2, 3, 4
TOOL = "paper_2508_19373_b200"
VERSION = "0.1.0"
B200_CFG = Path(__file__).resolve().parent / "presets" / "b200.cfg"


class ConfigFail(Exception):
    pass


def _block_config(args) -> BlockConfig:
    mp = import_moeplan()
    if args.model:
        from moeplan.configio import load_config, model_from_sections

        spec = model_from_sections(load_config(args.model), args.model)
        return BlockConfig.from_model_spec(spec)
    name = args.preset or "mixtral-8x7b"
    try:
        return get_config(name)
    except ValueError:
        try:
            return BlockConfig.from_model_spec(mp.load_preset(name))
        except Exception as exc:
            raise ConfigFail(str(exc)) from exc


def _hardware(args):
    """The B200 HardwareProfile from a reference-format [hardware] file."""
    from moeplan.configio import hardware_from_sections, load_config

    path = args.hw or str(B200_CFG)
    return hardware_from_sections(load_config(path), path, n_devices_override=args.devices)


def _manifest(args, t0: float, extra: Optional[Dict] = None) -> Dict:
    flags = {k: v for k, v in sorted(vars(args).items()) if k not in ("command", "func") and v is not None}
    m = {"tool": TOOL, "version": VERSION, "command": args.command, "flags": flags,
         "seed": getattr(args, "seed", None), "preset": getattr(args, "preset", None),
         "config_paths": {"model": getattr(args, "model", None), "hw": getattr(args, "hw", None) or str(B200_CFG)},
         "wall_s": time.perf_counter() - t0}
    m.update(extra or {})
    return m


def _plan_dict(plan) -> Dict:
    return {"attention": plan.attention.label(), "expert_prefill": plan.expert_prefill.label(),
            "expert_decode": plan.expert_decode.label(), "predicted_total_s": plan.predicted_total_s}


def cmd_plan(args) -> Dict:
    from .plan import calibrated_plan, plan_for

    mp = import_moeplan()
    cfg = _block_config(args)
    hw = _hardware(args)
    t = time.perf_counter()
    if args.calibrated:
        res, src = calibrated_plan(cfg, hw.n_devices, args.batch, args.input_len, args.output_len, hw=hw)
    else:
        res, src = plan_for(cfg, hw.n_devices, args.batch, args.input_len, args.output_len, hw=hw), "roofline"
    solve_s = time.perf_counter() - t
    out = {"model": cfg.name, "n_devices": hw.n_devices, "plan": _plan_dict(res.plan), "cost_source": src,
           "solver_wall_s": solve_s}
    try:
        k, i, j = mp.baseline_indices(res.catalog, "tp")
        out["baseline_tp"] = {"attention": res.catalog.attention[k].label(),
                              "expert_prefill": res.catalog.expert[i].label(),
                              "expert_decode": res.catalog.expert[j].label()}
    except Exception as exc:  # e.g. no pure-TP attention for this model at N
        out["baseline_tp"] = f"unavailable: {exc}"
    return out


def cmd_measure(args) -> Dict:
    from . import calib

    cfg = _block_config(args)
    n = args.devices or 1
    stages = tuple(args.stage) if args.stage else None
    meas = calib.measure_catalog(cfg, n, args.batch, args.input_len, args.output_len, reps=args.reps,
                                 stages=stages)
    samples = calib.to_samples(meas)
    out_csv = args.out_csv
    from moeplan.costmodel import write_samples_csv

    write_samples_csv(samples, out_csv)
    return {"model": cfg.name, "n_devices": n, "samples_csv": out_csv, "n_samples": len(samples),
            "cells": [{"module": m.module, "stage": m.stage, "strategy": m.strategy,
                       "measured_us": m.measured_s * 1e6, "roofline_us": m.roofline_s * 1e6, "eta": m.eta}
                      for m in meas]}


def cmd_run(args) -> Dict:
    import torch

    from .executor import HapMoEBlock, KVCache
    from .plan import plan_for

    cfg = _block_config(args)
    res = plan_for(cfg, 1, args.batch, args.input_len, args.output_len)
    out = {"model": cfg.name, "plan": _plan_dict(res.plan)}
    g = torch.Generator(device="cuda")
    g.manual_seed(args.seed)
    blk = HapMoEBlock.from_plan(cfg, res.plan, "prefill", seed=args.seed)
    T = args.batch * args.input_len
    x = torch.randn(T, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / args.steps

    ms = timed(lambda: blk.forward(x, "prefill", args.batch, args.input_len))
    out["prefill"] = {"tokens": T, "ms": ms, "tokens_per_s": T / ms * 1e3}
    if args.output_len > 0:
        kv = args.input_len + args.output_len // 2  # planner.py:226
        cache = KVCache.empty(args.batch, cfg.n_kv_heads, kv, cfg.head_dim, "cuda", random=True)
        pos = torch.full((args.batch,), kv - 1, device="cuda", dtype=torch.int32)
        xd = torch.randn(args.batch, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
        bd = HapMoEBlock.from_plan(cfg, res.plan, "decode", seed=args.seed)
        graph, _ = bd.capture_graph(xd, "decode", args.batch, kv_cache=cache, positions=pos)
        ms_d = timed(graph.replay)
        out["decode"] = {"batch": args.batch, "kv_len": kv, "ms": ms_d, "tokens_per_s": args.batch / ms_d * 1e3}
    return out


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog=TOOL, description=__doc__.split("\n\n")[0])
    p.add_argument("--version", action="version", version=f"{TOOL} {VERSION}")
    sub = p.add_subparsers(dest="command", required=True)

    def common(sp, hw=True):
        sp.add_argument("--preset", help="model preset (moeplan presets + mixtral-8x22b, tiny)")
        sp.add_argument("--model", help="model config file ([model] section, reference format)")
        if hw:
            sp.add_argument("--hw", help="hardware config file ([hardware] section); default presets/b200.cfg")
        sp.add_argument("--devices", type=int, help="device count (overrides the hardware file)")
        sp.add_argument("--batch", type=int, default=8)
        sp.add_argument("--input", type=int, default=2048, dest="input_len")
        sp.add_argument("--output-len", type=int, default=0)
        sp.add_argument("--seed", type=int, default=0)

    sp = sub.add_parser("plan", help="reference ILP plan on B200")
    common(sp)
    sp.add_argument("--calibrated", action="store_true", help="use the B200-measured module tables")
    sp.set_defaults(func=cmd_plan)
    sp = sub.add_parser("measure", help="write the reference calibration CSV from B200 measurements")
    common(sp, hw=False)
    sp.add_argument("--stage", action="append", choices=("prefill", "decode"))
    sp.add_argument("--reps", type=int, default=5)
    sp.add_argument("--out-csv", required=True)
    sp.set_defaults(func=cmd_measure)
    sp = sub.add_parser("run", help="time the planned block forward on this GPU")
    common(sp, hw=False)
    sp.add_argument("--steps", type=int, default=10)
    sp.set_defaults(func=cmd_run)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    t0 = time.perf_counter()
    mp = import_moeplan()
    from moeplan.arch import SpecError
    from moeplan.configio import ConfigError

    try:
        payload = args.func(args)
    except (ConfigFail, ConfigError, SpecError, FileNotFoundError, ValueError) as exc:
        print(json.dumps({"error": "config", "detail": str(exc)}), file=sys.stderr)
        return EXIT_CONFIG
    except mp.InfeasibleError as exc:
        print(json.dumps({"error": "infeasible", "detail": str(exc)}), file=sys.stderr)
        return EXIT_INFEASIBLE
    except Exception as exc:  # invariant breach / device failure
        print(json.dumps({"error": "internal", "detail": f"{type(exc).__name__}: {exc}"}), file=sys.stderr)
        return EXIT_INTERNAL
    payload["manifest"] = _manifest(args, t0)
    print(json.dumps(payload, indent=1, default=str))
    return EXIT_OK
