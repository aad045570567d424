#!/usr/bin/env python
"""HAP MoE-block benchmark on B200 (contract: see DESIGN.md §Measurement).

Workload (BASELINE.json configs[1]): one Mixtral-8x7B MoE decoder block,
bf16, prefill 8 x 2048 tokens (the headline ``value``) and decode batch 64 at
kv length 2048 (``decode``), for the plan the reference ILP picks on this
many B200s (``moeplan.plan``) and for the reference's pure-TP plan
(``baseline_indices(catalog, "tp")``).  A step = one forward of the block
over the whole global batch; scaling is strong (fixed global batch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mixtral-8x7B MoE-block tokens/s at 1/2/4/8 B200, HAP plan vs pure TP"
PREFILL_BATCH, PREFILL_SEQ = 8, 2048
DECODE_BATCH, DECODE_KV = 64, 2048


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------ clock sampler --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ distributed --
def dist_setup(n_gpus: int):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    if world > 1:
        # HAP_DIST_BACKEND=gloo: validation mode for the multi-rank path on a
        # single GPU (ranks share the device, collectives staged through host
        # memory; the numbers are not scaling measurements).  NCCL otherwise.
        backend = os.environ.get("HAP_DIST_BACKEND", "nccl")
        dev = local % torch.cuda.device_count() if backend == "gloo" else local
        torch.cuda.set_device(dev)
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def physical_gpu(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            return int(vis.split(",")[local])
        except (ValueError, IndexError):
            return local
    return local


def max_over_ranks(v: float) -> float:
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return v


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ---------------------------------------------------------------- workloads --
def global_input(cfg, tokens: int, seed: int):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn(tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)


def local_slice(x, block, batch: int, seq: int):
    from paper_2508_19373_b200.layout import replica_sequences

    s0, s1 = replica_sequences(batch, block.deg.a_dp, block.lay.a_rep)
    return x[s0 * seq:s1 * seq].contiguous()


TIMED_LAUNCHES = {}


def time_loop(fn, steps: int, warmup: int, tag: str = "", finish=None):
    """Device time per step (CUDA events on the launching stream, max over ranks).
    finish(): joins side streams into the launching stream before the end event."""
    import torch

    from paper_2508_19373_b200 import ops as K

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    l0 = K.LAUNCHES[0]
    s.record()
    for _ in range(steps):
        fn()
    if finish is not None:
        finish()
    e.record()
    torch.cuda.synchronize()
    TIMED_LAUNCHES[tag] = K.LAUNCHES[0] - l0
    barrier()
    ms = s.elapsed_time(e)
    return max_over_ranks(ms) / steps


def bench_prefill(block, cfg, steps, warmup, x_global):
    x = local_slice(x_global, block, PREFILL_BATCH, PREFILL_SEQ)
    return time_loop(lambda: block.forward(x, "prefill", PREFILL_BATCH, PREFILL_SEQ), steps, warmup,
                     tag=f"prefill:{block.deg.label()}")


def make_decode_state(block, cfg):
    import torch

    from paper_2508_19373_b200.executor import KVCache
    from paper_2508_19373_b200.layout import replica_sequences

    s0, s1 = replica_sequences(DECODE_BATCH, block.deg.a_dp, block.lay.a_rep)
    nb = s1 - s0
    cache = KVCache.empty(max(nb, 1), block.w.n_kv_local, DECODE_KV, cfg.head_dim, "cuda", random=True)
    pos = torch.full((nb,), DECODE_KV - 1, device="cuda", dtype=torch.int32)
    x = global_input(cfg, DECODE_BATCH, seed=7)[s0:s1].contiguous()
    return x, cache, pos


DECODE_MIN_STEPS = 200  # a decode step is ~0.65 ms: time >= 130 ms of replays, after 20 warm-up steps


def bench_decode(block, cfg, steps, warmup):
    """Decode step timing; single-device non-EP plans replay a CUDA graph of the
    block (the step is launch-bound at B=64), others run eagerly.  The loop runs
    max(steps, DECODE_MIN_STEPS) steps so the clocks settle (the headline prefill
    loop keeps the contract's K)."""
    x, cache, pos = make_decode_state(block, cfg)
    steps, warmup = max(steps, DECODE_MIN_STEPS), max(warmup, 20)
    if block.graph_capturable(DECODE_BATCH):
        g, _ = block.capture_graph(x, "decode", DECODE_BATCH, kv_cache=cache, positions=pos)
        return time_loop(g.replay, steps, warmup), "cuda_graph"
    return time_loop(lambda: block.forward(x, "decode", DECODE_BATCH, kv_cache=cache, positions=pos,
                                           max_position=DECODE_KV - 1), steps, warmup), "eager"


def bench_peer_variant(cfg, hap_p, hap_d, rank, weights, x_global, steps, warmup):
    """N > 1: the HAP plan again with every exchange that has a peer-memory form
    switched to it (EP dispatch/combine planned on the device, the DP<->TP
    boundary pushed by the norm / combine, one-shot decode all-reduces).  These
    paths are opt-in in the executor until timed on an NVLink box; this is that
    timing.  Barrier waits trap after ~20 s rather than hang, so a failure here
    is reported in the line instead of stalling the run."""
    from paper_2508_19373_b200.executor import HapMoEBlock

    out = {}
    blocks = []
    try:
        for stage, sp in (("prefill", hap_p), ("decode", hap_d)):
            blk = HapMoEBlock(cfg, sp.degrees, None, rank=rank, weights=weights)
            blocks.append(blk)
            blk.ep_peer = blk.boundary_peer = True
            if blk.comm is not None:
                blk.comm.enable_peer_allreduce(["attn_tp_group", "exp_tp_group"])
            if stage == "prefill":
                ms = bench_prefill(blk, cfg, steps, warmup, x_global)
                out.update({"plan": sp.label(), "prefill_ms": ms,
                            "prefill_tokens_per_s": PREFILL_BATCH * PREFILL_SEQ / (ms / 1e3)})
            else:
                ms, mode = bench_decode(blk, cfg, steps, warmup)
                out.update({"decode_plan": sp.label(), "decode_ms": ms, "decode_mode": mode,
                            "decode_tokens_per_s": DECODE_BATCH / (ms / 1e3)})
    except Exception as exc:  # noqa: BLE001 - reported in the JSON line
        out["error"] = f"{type(exc).__name__}: {str(exc)[:300]}"
    for b in blocks:
        try:
            b.close()
        except Exception:  # noqa: BLE001
            pass
    return out


def decode_bytes(cfg, block_routing_idx) -> float:
    """Algorithmic HBM bytes of one decode step over the whole job."""
    import torch

    touched = int(torch.unique(block_routing_idx).numel())
    h, I, kv = cfg.hidden, cfg.inter, cfg.kv_dim
    experts = touched * 3 * h * I * 2 + cfg.n_shared * 3 * h * I * 2
    attn_w = 2 * (h * h + h * kv) * 2
    kv_bytes = DECODE_BATCH * DECODE_KV * 2 * kv * 2
    router = cfg.n_experts * h * 2
    return float(experts + attn_w + kv_bytes + router)


# ------------------------------------------------------------------- CPU side --
def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_setup(cfg, sample_tokens: int):
    """The oracle port of the block (numpy fp32 matmuls on every host core, the
    BASELINE.md §3 plan) on a bounded prefill sample."""
    import numpy as np

    from oracle import moe_block as O

    O.set_precision("f32")
    spec = _oracle_spec(cfg)
    W = _oracle_weights(cfg)
    x = np.random.default_rng(1).standard_normal((sample_tokens, cfg.hidden)).astype(np.float32)
    return lambda: O.block_forward(spec, W, x, 1)


def _oracle_spec(cfg):
    from oracle import moe_block as O

    return O.BlockSpec(hidden=cfg.hidden, n_q_heads=cfg.n_q_heads, n_kv_heads=cfg.n_kv_heads,
                       head_dim=cfg.head_dim, n_experts=cfg.n_experts, top_k=cfg.top_k, inter=cfg.inter,
                       n_shared=cfg.n_shared, norm_topk_prob=cfg.norm_topk_prob, qkv_bias=cfg.qkv_bias,
                       rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)


_ORACLE_W = {}


def _oracle_weights(cfg):
    from oracle import moe_block as O

    if cfg.name not in _ORACLE_W:
        _ORACLE_W[cfg.name] = O.random_weights(_oracle_spec(cfg), seed=0, bf16=False)
    return _ORACLE_W[cfg.name]


def cpu_decode_baseline(cfg, batch: int = DECODE_BATCH, kv: int = DECODE_KV):
    """One full-size decode step (B=64 @ kv 2048) of the oracle port, fp32, all host cores."""
    import numpy as np

    from oracle import moe_block as O

    O.set_precision("f32")
    spec = _oracle_spec(cfg)
    W = _oracle_weights(cfg)
    rng = np.random.default_rng(7)
    kc = rng.standard_normal((batch, cfg.n_kv_heads, kv, cfg.head_dim), dtype=np.float32)
    vc = rng.standard_normal((batch, cfg.n_kv_heads, kv, cfg.head_dim), dtype=np.float32)
    x = rng.standard_normal((batch, cfg.hidden), dtype=np.float32)
    pos = np.full(batch, kv - 1)
    O.decode_forward(spec, W, x, kc, vc, pos)
    t0 = time.perf_counter()
    O.decode_forward(spec, W, x, kc, vc, pos)
    dt = time.perf_counter() - t0
    return {"value": batch / dt, "unit": "tokens/s", "ms_per_step": dt * 1e3, "cores": cpu_cores(),
            "sample": f"one {cfg.name} decode step B={batch} @ kv {kv} through oracle decode_forward (fp32)"}


def planner_baseline(cfg, world: int, reps: int = 20):
    """The reference's own CPU path on this workload:
    moeplan plan() for the prefill and decode scenarios, roofline tables and
    the B200-measured tables, median of `reps` calls on the host."""
    from paper_2508_19373_b200.plan import calibrated_plan, plan_for

    out = {}
    for name, args in (("prefill_8x2048", (PREFILL_BATCH, PREFILL_SEQ, 0)),
                       ("decode_b64", (DECODE_BATCH, DECODE_KV // 2, DECODE_KV))):
        for kind, fn in (("roofline", plan_for), ("measured_tables", calibrated_plan)):
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn(cfg, world, *args)
                ts.append(time.perf_counter() - t0)
            out[f"{name}_{kind}_ms"] = statistics.median(ts) * 1e3
    out.update({"reps": reps, "cores": 1, "what": "moeplan.plan / solve_ilp on the host (reference CPU path), "
                                                  "median of reps"})
    return out


def cpu_baseline(cfg, sample_tokens: int, reps: int = 2, decode: bool = True):
    fn = cpu_reference_setup(cfg, sample_tokens)
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps
    out = {"value": sample_tokens / dt, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
           "sample": f"oracle/moe_block.py block_forward (numpy fp32 matmuls on all host cores, {cfg.name} full "
                     f"dims), 1 sequence x {sample_tokens} tokens prefill, mean of {reps}"}
    if decode:
        out["decode"] = cpu_decode_baseline(cfg)
    out["planner"] = planner_baseline(cfg, 8)  # the 8-GPU plan search the reference exists for
    return out


def run_reference(args):
    """--impl reference: the reference-side CPU path for this metric (the oracle port; the
    reference package has no forward implementation)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2508_19373_b200.config import get_config

    cfg = get_config(args.config)
    # keep the whole --steps/--warmup run within a few minutes: shrink the per-step
    # sample when many steps are requested (tokens/s is per-token work, so the
    # sample size does not change the metric beyond fixed per-call overheads)
    n_calls = args.steps + args.warmup
    args.cpu_sample_tokens = int(max(32, min(args.cpu_sample_tokens, 256 * 23 // max(n_calls, 1))))
    fn = cpu_reference_setup(cfg, args.cpu_sample_tokens)
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    dt = (time.perf_counter() - t0) / args.steps
    val = args.cpu_sample_tokens / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} MoE block prefill (bounded CPU sample)", "model": cfg.name,
                   "global_batch": 1, "seq_len": args.cpu_sample_tokens, "parallelism": "host cores"},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
                         "sample": f"1 x {args.cpu_sample_tokens} tokens per step through oracle/moe_block.py (numpy fp32, all host cores)"},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-tp", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--peer", action="store_true",
                    help="N>1: also time the HAP plan with its peer-memory exchanges (CUDA IPC + device barriers). "
                         "Opt-in: validated only with ranks sharing one B200; a device-side barrier trap on a real "
                         "NVLink box would poison the CUDA context and cost the NCCL numbers of the same run")
    ap.add_argument("--no-peer", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-sample-tokens", type=int, default=256)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    from paper_2508_19373_b200 import ops as K
    from paper_2508_19373_b200.config import get_config
    from paper_2508_19373_b200.executor import HapMoEBlock
    from paper_2508_19373_b200.plan import baseline_plan, calibrated_plan, plan_for, stage_plan
    from paper_2508_19373_b200.weights import synthetic_weights

    rank, world, local = dist_setup(args.gpus)
    cfg = get_config(args.config)
    peaks = load_peaks()

    t_plan = time.perf_counter()
    res_roof = plan_for(cfg, world, PREFILL_BATCH, PREFILL_SEQ, 0)
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    # HAP plan = the reference ILP on B200-measured module tables (profiles/r01_calibration.json,
    # scripts/calibrate.py); falls back to the roofline plan when the scenario is not calibrated.
    res_p, plan_src = calibrated_plan(cfg, world, PREFILL_BATCH, PREFILL_SEQ, 0)
    res_d, _ = calibrated_plan(cfg, world, DECODE_BATCH, DECODE_KV // 2, DECODE_KV)  # kv = in + out//2
    hap_p, hap_d = stage_plan(res_p, "prefill"), stage_plan(res_d, "decode")
    plans = {"hap": (hap_p, hap_d)}
    roof_p = stage_plan(res_roof, "prefill")
    if world > 1 and roof_p.degrees != hap_p.degrees and not args.no_tp:
        plans["hap_roofline"] = (roof_p, hap_d)
    if world > 1 and not args.no_tp:
        try:
            plans["tp"] = (baseline_plan(res_p, "tp", "prefill"), baseline_plan(res_d, "tp", "decode"))
        except Exception as exc:  # e.g. Qwen2-57B at N=8 has no pure-TP attention
            plans["tp_unavailable"] = str(exc)

    weights = synthetic_weights(cfg, "cuda", seed=0)
    x_global = global_input(cfg, PREFILL_BATCH * PREFILL_SEQ, seed=1)
    blocks = {}

    def get_block(sp):
        key = sp.degrees
        if key not in blocks:
            blocks[key] = HapMoEBlock(cfg, key, None, rank=rank, weights=weights)
        return blocks[key]

    sampler = ClockSampler(physical_gpu(torch.cuda.current_device()))
    sampler.start()
    results = {}
    launches0 = K.LAUNCHES[0]
    for name, val in plans.items():
        if not isinstance(val, tuple):
            continue
        sp_p, sp_d = val
        blk = get_block(sp_p)
        ms_p = bench_prefill(blk, cfg, args.steps, args.warmup, x_global)
        r = {"plan": sp_p.label(), "prefill_ms": ms_p,
             "prefill_tokens_per_s": PREFILL_BATCH * PREFILL_SEQ / (ms_p / 1e3)}
        if not args.no_decode:
            bd = get_block(sp_d)
            ms_d, mode = bench_decode(bd, cfg, args.steps, args.warmup)
            r.update({"decode_plan": sp_d.label(), "decode_ms": ms_d, "decode_mode": mode,
                      "decode_steps": max(args.steps, DECODE_MIN_STEPS),
                      "decode_tokens_per_s": DECODE_BATCH / (ms_d / 1e3)})
        results[name] = r
    total_launches = K.LAUNCHES[0] - launches0
    clocks = sampler.stop()

    # -- whole-block roofline per plan: the reference's FLOP model (arch.py:145-178)
    # with the causal half of the score/value term removed, over N GPUs at the
    # measured dense bf16 peak
    from paper_2508_19373_b200.config import import_moeplan

    mpl = import_moeplan()
    spec = cfg.to_model_spec()
    T_pf = PREFILL_BATCH * PREFILL_SEQ
    f_attn = mpl.attention_flops(spec, T_pf, PREFILL_SEQ)
    f_useful = f_attn - 2 * T_pf * PREFILL_SEQ * cfg.hidden + mpl.expert_flops(spec, T_pf)
    roof_ms = f_useful / (world * peaks["bf16_tflops"] * 1e12) * 1e3
    for r in results.values():
        r["roofline_ms"] = roof_ms
        r["frac_of_roofline"] = roof_ms / r["prefill_ms"]
    roofline_block = {"flops_per_step": f_useful, "peak_tflops_per_gpu": peaks["bf16_tflops"], "n_gpus": world,
                      "ms": roof_ms, "frac": roof_ms / results["hap"]["prefill_ms"],
                      "convention": "attention_flops + expert_flops (reference arch.py:145-178), causal score/value "
                                    "term halved; measured burst bf16 peak"}

    # -- roofline of the dominant kernel (expert gate/up grouped GEMM), live CUDA events
    blk = get_block(hap_p)
    blk.timers = {}
    x = local_slice(x_global, blk, PREFILL_BATCH, PREFILL_SEQ)
    for _ in range(3):
        blk.forward(x, "prefill", PREFILL_BATCH, PREFILL_SEQ)
    torch.cuda.synchronize()
    blk.timers = {}
    for _ in range(args.steps):
        blk.forward(x, "prefill", PREFILL_BATCH, PREFILL_SEQ)
    torch.cuda.synchronize()
    gu = [s.elapsed_time(e) for s, e in blk.timers["gate_up"]]
    dn = [s.elapsed_time(e) for s, e in blk.timers["down"]]
    phase_ms = {k: statistics.mean(s.elapsed_time(e) for s, e in v) for k, v in blk.timers.items()}
    blk.timers = None
    gu_ms = max_over_ranks(statistics.mean(gu))
    dn_ms = max_over_ranks(statistics.mean(dn))
    T = PREFILL_BATCH * PREFILL_SEQ
    il = blk.w.inter_local
    # algorithmic FLOPs of one gate/up launch on this rank: rows routed here x 2*I_l x h x 2
    rows_here = int(blk.last_routing[2][-1].item()) if hap_p.degrees.e_ep == 1 else None
    if rows_here is None:
        rows_here = T * cfg.top_k // world
    gu_flops = 2.0 * rows_here * 2 * il * cfg.hidden
    dn_flops = 2.0 * rows_here * il * cfg.hidden
    achieved = gu_flops / (gu_ms / 1e3) / 1e12
    # DRAM traffic of the same launch from the newest committed ncu --set full capture
    # (profiles/<round>_gemm_traffic.json, written by scripts/summarize_profiles.py)
    traffic, traffic_src, traffic_ratio = None, None, None
    caps = sorted((ROOT / "profiles").glob("r*_gemm_traffic.json"))
    if caps:
        try:
            tj = json.loads(caps[-1].read_text())
            traffic = tj["gate_up"]["dram_bytes_per_launch"]
            traffic_ratio = tj["gate_up"]["traffic_over_algorithmic"]
            traffic_src = f"profiles/{caps[-1].name}"
        except Exception:
            traffic = None
    roofline = {"kernel": "hap::gemm::grouped_gemm_kernel (expert gate/up, SwiGLU epilogue)", "bound": "tensor",
                "achieved": achieved, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16_tflops_sustained"], "peak_kind": f"{peaks['source']} sustained",
                "frac_of_burst_peak": achieved / peaks["bf16_tflops"], "traffic": traffic,
                "traffic_over_algorithmic_bytes": traffic_ratio, "traffic_source": traffic_src,
                "algorithmic_flops_per_launch": gu_flops, "launch_ms": gu_ms,
                "down_proj": {"launch_ms": dn_ms, "achieved": dn_flops / (dn_ms / 1e3) / 1e12},
                "expert_gemms_share_of_step": (gu_ms + dn_ms) / results["hap"]["prefill_ms"]}

    # -- every kernel phase of the prefill step against its roofline (N=1: the
    # algorithmic work per launch below is for the whole, unsharded block)
    kernels = None
    if world == 1:
        T, h, d = PREFILL_BATCH * PREFILL_SEQ, cfg.hidden, cfg.head_dim
        nq, nkv, E, k = cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.top_k
        work = {  # phase: (algorithmic work per launch, bound)
            "norm": (2.0 * T * h * 2, "hbm"),
            "qkv": (2.0 * T * h * (nq + 2 * nkv) * d, "tensor"),
            "attn": (4.0 * T * PREFILL_SEQ * nq * d / 2, "tensor"),  # arch.py:161, causal half
            "o_proj": (2.0 * T * nq * d * h, "tensor"),
            "router": (T * h * 2.0 + E * h * 2.0 + T * k * 8.0, "hbm"),
            "permute": (T * h * 2.0 + T * k * h * 2.0 + T * k * 4.0, "hbm"),
            "gate_up": (gu_flops, "tensor"),
            "down": (dn_flops, "tensor"),
            "combine": (T * k * h * 2.0 + 2.0 * T * h * 2, "hbm"),
        }
        kernels = {}
        for name, (wk, bound) in work.items():
            if name not in phase_ms:
                continue
            ms = phase_ms[name]
            if bound == "tensor":
                ach, peak, unit = wk / (ms / 1e3) / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s"
            else:
                ach, peak, unit = wk / (ms / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s"
            kernels[name] = {"ms": ms, "bound": bound, "work": wk, "achieved": ach, "peak": peak, "unit": unit,
                             "frac": ach / peak}
            if bound == "hbm":  # the north star's ~8 TB/s denominator beside the measured copy peak
                kernels[name]["frac_of_8TBps"] = ach / 8000.0

    # -- decode HBM roofline (whole step)
    decode = None
    if not args.no_decode:
        bd = get_block(hap_d)
        xd, cache, pos = make_decode_state(bd, cfg)
        bd.forward(xd, "decode", DECODE_BATCH, kv_cache=cache, positions=pos)
        torch.cuda.synchronize()
        dbytes = decode_bytes(cfg, bd.last_routing[0])
        ms_d = results["hap"]["decode_ms"]
        gbs = dbytes / (ms_d / 1e3) / 1e9
        decode = {"workload": f"{cfg.name} block decode B={DECODE_BATCH} kv={DECODE_KV}", "plan": hap_d.label(),
                  "tokens_per_s": results["hap"]["decode_tokens_per_s"], "ms_per_step": ms_d,
                  "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"] * world, "unit": "GB/s",
                               "frac": gbs / (peaks["hbm_gbs"] * world), "algorithmic_bytes_per_step": dbytes,
                               "frac_of_8TBps": gbs / (8000.0 * world)}}

    # -- e2e through the public API with host buffers (pinned), H2D + D2H in the timed region
    x_loc = local_slice(x_global, blk, PREFILL_BATCH, PREFILL_SEQ)
    x_host = x_loc.cpu().pin_memory()
    out_host = torch.empty_like(x_host).pin_memory()

    # every step copies its input from pinned host memory and its output back;
    # forward_host double-buffers across steps (H2D of step i+1 and D2H of
    # step i-1 overlap step i's forward), the way a serving loop streams batches
    def e2e_step():
        blk.forward_host(x_host, out_host, PREFILL_BATCH, PREFILL_SEQ)
    e2e_finish = blk.host_sync
    api = ("paper_2508_19373_b200.executor.HapMoEBlock.forward_host (pinned host in/out every step; "
           "H2D(i+1) and D2H(i-1) overlap forward(i); the timed region ends after the last D2H)")

    e2e_ms = time_loop(e2e_step, args.steps, args.warmup, finish=e2e_finish)
    h2d = x_host.numel() * 2 * world
    e2e = {"value": T / (e2e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": h2d, "api": api}

    # N > 1, last (its failure must not cost the other numbers): the HAP plan over peer memory
    peer = None
    if world > 1 and args.peer and not args.no_peer:
        peer = bench_peer_variant(cfg, hap_p, hap_d, rank, weights, x_global, args.steps, args.warmup)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_sample_tokens)

    if rank == 0:
        hap = results["hap"]
        line = {
            "metric": METRIC, "value": hap["prefill_tokens_per_s"], "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": hap["prefill_ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: random-init weights N(0,0.02) bf16, x ~ N(0,1)",
            "config": {"workload": f"{cfg.name} MoE decoder block (attention + experts), bf16 prefill "
                                   f"{PREFILL_BATCH}x{PREFILL_SEQ}",
                       "model": cfg.name, "global_batch": PREFILL_BATCH, "seq_len": PREFILL_SEQ,
                       "parallelism": hap["plan"],
                       "planner": f"moeplan solve_ilp (reference ILP) on {plan_src}",
                       "planner_ms": plan_ms,
                       "l2": "no flush: every step streams > L2 (2.8 GB expert weights + 128 MB activations)"},
            "plans": results, "hap_peer_exchanges": peer, "decode": decode, "roofline": roofline,
            "roofline_block": roofline_block,
            "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": TIMED_LAUNCHES.get(f"prefill:{hap_p.degrees.label()}"),
            "gpu_launches_note": "kernels of libhap_kernels.so launched in the headline timed region (this rank)",
            "gpu_launches_all_bench_loops": total_launches,
            "clocks": clocks, "peaks": peaks,
        }
        print(json.dumps(line), flush=True)
    for b in blocks.values():
        b.close()
    barrier()
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
