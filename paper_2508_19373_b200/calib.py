"""B200 recalibration of the reference latency models.

The reference prices a plan with per-layer compute terms
``t = flops / peak * eta(b, s, h)`` for the attention module (rows
``(ceil(B/A_d), S or 1, h)``, flops ``attention_flops / A_t``) and the
expert module (rows ``(B, S or 1, h)``, flops ``expert_flops * gamma / N``)
(planner.py:222-250), and communication terms ``volume / bw * rho``
(planner.py:182-195).  Its calibration interface is ``CalibrationSample``
-> ``train_forest`` -> ``CostModels(eta, rho)`` (costmodel.py:40-161,
planner.py:57-62).

This module measures, on one B200, the per-device time of the attention and
expert modules for EVERY strategy of the reference catalog (each rank's
shard: heads / A_t and ceil(B/A_d) sequences; experts E/ep with the rows the
routing actually sends there, intermediate slice I/tp) using the product
kernels, then

1. feeds them through the reference API unchanged: one compute
   ``CalibrationSample`` per measurement with ``context = peak * 2bsh^2 /
   flops`` so that the sample's target equals measured * peak / flops, the
   eta the planner multiplies onto ``flops / peak`` (SURVEY.md §7 hard part
   6, "context trick"); ``train_forest`` fits eta; ``plan(..,
   CostModels(eta=...))`` re-plans;
2. reports the held-out predicted-vs-measured error of that eta model, and
   the collision error the reference's (b, s, h)-only feature set imposes
   (attention and expert rows that share features but not efficiency);
3. provides the additive per-module extension ``measured_cost_tensors``:
   the reference's CostTensors with t_a / t_e replaced by the measured
   per-strategy times (communication and switch costs unchanged), solved by
   the reference's own ``solve_ilp``.

Collective (rho) samples need >= 2 GPUs: ``measure_collectives`` runs under
torchrun and emits communication samples in the same CSV format.
"""

from __future__ import annotations

import math
import statistics
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import ops as K
from .config import B200_PEAK_FLOPS, BlockConfig, b200_hardware, import_moeplan
from .weights import swiglu_half_width

BF16 = torch.bfloat16


def _events_time(fn, reps: int, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return statistics.median(ts)


def _graph_time(fn, reps: int, warmup: int = 2) -> float:
    """Time fn as CUDA-graph replays — how the executor runs a decode step, so a
    decode cell carries no per-launch host overhead the model does not pay."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    t = _events_time(g.replay, reps, warmup=warmup)
    del g
    return t


def _stage_time(fn, stage: str, reps: int) -> float:
    return _graph_time(fn, reps) if stage == "decode" else _events_time(fn, reps)


def _rand(shape, std=1.0):
    t = torch.randn(shape, device="cuda", dtype=BF16)
    return t.mul_(std) if std != 1.0 else t


# ------------------------------------------------------------- attention --
def measure_attention(cfg: BlockConfig, tp: int, b_rep: int, S: int, stage: str, kv_len: int = 2048,
                      reps: int = 5) -> float:
    """Per-device attention-module time of one rank under attention (tp, dp):
    rmsnorm -> QKV GEMM + RoPE -> attention core -> O GEMM (+residual)."""
    h, d = cfg.hidden, cfg.head_dim
    nq, nkv = cfg.n_q_heads // tp, cfg.n_kv_heads // tp
    T = b_rep * S if stage == "prefill" else b_rep
    x = _rand((T, h))
    ln = torch.ones(h, device="cuda", dtype=BF16)
    wqkv = _rand(((nq + 2 * nkv) * d, h), 0.02)
    bqkv = _rand(((nq + 2 * nkv) * d,), 0.02) if cfg.qkv_bias else None
    wo = _rand((h, nq * d), 0.02)
    attn = torch.empty(T, nq * d, device="cuda", dtype=BF16)
    if stage == "prefill":
        pos = torch.arange(S, device="cuda", dtype=torch.int32).repeat(b_rep)

        def fn():
            xn = K.rmsnorm(x, ln, cfg.rms_eps)
            qkv = K.gemm_qkv_rope(xn, wqkv, pos, nq + nkv, d, cfg.rope_theta, bias=bqkv)
            K.attn_prefill(qkv, nq, nkv, d, b_rep, S, attn)
            K.gemm(attn, wo, residual=x)
    else:
        pos = torch.full((T,), kv_len - 1, device="cuda", dtype=torch.int32)
        kc = _rand((T, nkv, kv_len, d))
        vc = _rand((T, nkv, kv_len, d))
        ws = torch.empty(K.attn_decode_workspace_bytes(T, nq, d, kv_len), device="cuda", dtype=torch.uint8)

        def fn():
            xn = K.rmsnorm(x, ln, cfg.rms_eps)
            qkv = K.gemm_qkv_rope(xn, wqkv, pos, nq + nkv, d, cfg.rope_theta, bias=bqkv)
            K.attn_decode(qkv, kc, vc, pos, nq, nkv, d, attn, ws)
            K.gemm(attn, wo, residual=x)
    t = _stage_time(fn, stage, reps)
    del x, wqkv, wo, attn
    return t


# ---------------------------------------------------------------- experts --
def skewed_router(router: torch.Tensor, n_experts: int) -> torch.Tensor:
    """SURVEY §8(d) skewed-routing workload: router row e scaled by 1 + 0.1*e
    (expert E-1 is picked most), so EP groups receive unequal row counts."""
    scale = torch.ones(router.shape[0], 1, device=router.device, dtype=torch.float32)
    scale[:n_experts, 0] = 1.0 + 0.1 * torch.arange(n_experts, device=router.device, dtype=torch.float32)
    return (router.float() * scale).to(router.dtype)


def measure_experts(cfg: BlockConfig, tp: int, ep: int, dp: int, B: int, S: int, stage: str,
                    reps: int = 5, skew: bool = False, detail: Optional[dict] = None) -> float:
    """Per-device expert-module time of the slowest rank under expert (tp, ep, dp):
    router + permute over the rank's own token shard, grouped gate/up + down
    GEMMs over the rows the routing of its expert-DP replica's tokens
    (T / dp) sends to its E/ep experts (I/tp slice), shared expert, weighted
    combine.  The EP group measured is the one receiving the most rows (the
    reference charges EP a fixed gamma = 1.3 for this imbalance,
    planner.py:54, 243-248; here it is measured, and reported in
    detail["imbalance"] = max / mean rows over the EP groups).  skew: the
    skewed-routing workload (skewed_router).  Collectives excluded (priced by rho)."""
    h, E, k = cfg.hidden, cfg.n_experts, cfg.top_k
    T_all = B * S if stage == "prefill" else B
    n_shards = ep * dp
    T_own = max(1, math.ceil(T_all / n_shards)) if n_shards > 1 else T_all
    T_rep = max(1, math.ceil(T_all / dp)) if dp > 1 else T_all  # tokens of one expert-DP replica
    El = E // ep
    Il = cfg.inter // tp
    hw = swiglu_half_width(Il)
    x_all = _rand((T_all, h))
    router = _rand((E + (1 if cfg.n_shared else 0), h), 0.02)
    if skew:
        router = skewed_router(router, E)
    w13 = _rand((El, 2 * Il, h), 0.02)
    w2 = _rand((El, h, Il), 0.02)
    # routing of the replica's tokens -> rows received by the busiest EP group (untimed setup)
    x_rep = x_all[:T_rep].contiguous()
    idx_all = torch.empty(T_rep, k, device="cuda", dtype=torch.int32)
    tw_all = torch.empty(T_rep, k, device="cuda", dtype=torch.float32)
    sg_all = torch.empty(T_rep, device="cuda", dtype=torch.float32) if cfg.n_shared else None
    K.router_topk(x_rep, router, E, k, cfg.norm_topk_prob, bool(cfg.n_shared), idx_all, tw_all, sg_all)
    counts = torch.bincount(idx_all.view(-1).long(), minlength=E).cpu()
    group_rows = counts.view(ep, El).sum(1)
    g_max = int(torch.argmax(group_rows))
    if detail is not None:
        detail["group_rows"] = [int(r) for r in group_rows]
        detail["imbalance"] = float(group_rows.max()) / max(float(group_rows.float().mean()), 1e-9)
        detail["ep_group"] = g_max
    local = idx_all.view(-1).clone() - g_max * El
    local = torch.where((local >= 0) & (local < El), local, torch.full_like(local, -1))
    R_all = T_rep * k
    ws_all = torch.empty(max(K.permute_workspace_bytes(R_all, El), 16), device="cuda", dtype=torch.uint8)
    dst_all = torch.empty(R_all, device="cuda", dtype=torch.int32)
    seg_l = torch.empty(El + 1, device="cuda", dtype=torch.int32)
    K.moe_permute(local, El, None, k, None, dst_all, seg_l, ws_all)
    torch.cuda.synchronize()
    n_recv = int(seg_l[-1].item())
    x_recv = _rand((max(n_recv, 1), h))
    H = torch.empty(max(n_recv, 1), Il, device="cuda", dtype=BF16)
    Y = torch.empty(max(n_recv, 1), h, device="cuda", dtype=BF16)
    # own shard
    x_own = x_all[:T_own].contiguous()
    R = T_own * k
    idx = torch.empty(T_own, k, device="cuda", dtype=torch.int32)
    tw = torch.empty(T_own, k, device="cuda", dtype=torch.float32)
    sg = torch.empty(T_own, device="cuda", dtype=torch.float32) if cfg.n_shared else None
    x_perm = torch.empty(R, h, device="cuda", dtype=BF16)
    dst = torch.empty(R, device="cuda", dtype=torch.int32)
    seg = torch.empty(E + 1, device="cuda", dtype=torch.int32)
    ws = torch.empty(max(K.permute_workspace_bytes(R, E), 16), device="cuda", dtype=torch.uint8)
    y_back = _rand((R, h))
    out = torch.empty(T_own, h, device="cuda", dtype=BF16)
    ws13 = ws2 = None
    if cfg.n_shared:
        sil = cfg.shared_inter // tp
        hws = swiglu_half_width(sil)
        ws13 = _rand((2 * sil, h), 0.02)
        ws2 = _rand((h, sil), 0.02)

    def fn():
        K.router_topk(x_own, router, E, k, cfg.norm_topk_prob, bool(cfg.n_shared), idx, tw, sg)
        K.moe_permute(idx.view(-1), E, x_own, k, x_perm, dst, seg, ws)
        if n_recv:
            K.grouped_gemm(x_recv, w13, El, seg_l, H, swiglu_half=hw)
            K.grouped_gemm(H, w2, El, seg_l, Y)
        ys = None
        if cfg.n_shared:
            hs = K.gemm(x_own, ws13, swiglu_half=hws)
            ys = K.gemm(hs, ws2)
        K.moe_combine(y_back, dst, tw, T_own, k, out, residual=x_own, shared_y=ys, shared_gate=sg)
    t = _stage_time(fn, stage, reps)
    del x_all, x_rep, w13, w2, x_recv, H, Y
    torch.cuda.empty_cache()
    return t


# ------------------------------------------------------------ the catalog --
@dataclass
class Measurement:
    model: str
    n: int
    module: str          # "attention" | "experts"
    stage: str           # "prefill" | "decode"
    strategy: str
    index: int           # catalog index (k for attention, i for experts)
    b: float             # planner eta features (planner.py:169-170, 229-250)
    s: float
    h: float
    flops: float         # planner flop charge of this cell
    measured_s: float
    roofline_s: float
    imbalance: float = 1.0  # experts: measured max/mean EP-group rows (the reference's gamma)

    @property
    def eta(self) -> float:
        return self.measured_s / self.roofline_s


def measure_catalog(cfg: BlockConfig, n: int, batch: int, input_len: int, output_len: int,
                    reps: int = 5, gamma: float = 1.3, cache: Optional[dict] = None,
                    stages: Optional[Tuple[str, ...]] = None, skew: bool = False) -> List[Measurement]:
    """Measured per-device module time for every (strategy, stage) cell the
    planner prices for this scenario (build_cost_tensors, planner.py:222-250).
    Cells of stages not measured keep the planner's own estimate."""
    mp = import_moeplan()
    spec = cfg.to_model_spec()
    hw = b200_hardware(n)
    cat = mp.build_catalog(spec, hw)
    cache = {} if cache is None else cache
    decode_kv = max(1, input_len + output_len // 2)
    out: List[Measurement] = []
    if stages is None:
        stages = ("prefill",) + (("decode",) if output_len > 0 else ())
    for st in stages:
        for k_, a in enumerate(cat.attention):
            b_rep = math.ceil(batch / a.dp_degree)
            key = ("attn", cfg.name, a.tp_degree, b_rep, input_len, st, decode_kv)
            if key not in cache:
                cache[key] = measure_attention(cfg, a.tp_degree, b_rep, input_len, st, decode_kv, reps)
            if st == "prefill":
                fl = mp.attention_flops(spec, b_rep * input_len, input_len) / a.tp_degree
                s = input_len
            else:
                fl = mp.attention_flops(spec, b_rep, decode_kv) / a.tp_degree
                s = 1
            out.append(Measurement(cfg.name, n, "attention", st, a.label(), k_, b_rep, s, cfg.hidden, fl,
                                   cache[key], fl / hw.peak_flops))
        for i, e in enumerate(cat.expert):
            key = ("exp", cfg.name, e.tp_degree, e.ep_degree, e.dp_degree, batch, input_len, st, skew)
            if key not in cache:
                det = {}
                cache[key] = (measure_experts(cfg, e.tp_degree, e.ep_degree, e.dp_degree, batch, input_len, st,
                                              reps, skew=skew, detail=det), det.get("imbalance", 1.0))
            imb = gamma if e.ep_degree > 1 else 1.0
            tokens = batch * input_len if st == "prefill" else batch
            fl = mp.expert_flops(spec, tokens) * imb / n
            out.append(Measurement(cfg.name, n, "experts", st, e.label(), i, batch,
                                   input_len if st == "prefill" else 1, cfg.hidden, fl, cache[key][0],
                                   fl / hw.peak_flops, imbalance=cache[key][1]))
    return out


def to_samples(meas: List[Measurement], peak: float = B200_PEAK_FLOPS):
    """Reference CalibrationSamples (costmodel.py:40-82) whose target equals
    measured * peak / flops, i.e. the eta the planner applies to this cell."""
    mp = import_moeplan()
    return [mp.CalibrationSample(kind="compute", b=m.b, s=m.s, h=m.h,
                                 context=peak * 2.0 * m.b * m.s * m.h * m.h / m.flops,
                                 measured_latency=m.measured_s) for m in meas]


def fit_eta(meas: List[Measurement], seed: int = 0, holdout: float = 0.25):
    """train_forest on a seeded split; returns (model, train_err, test_err, test_rows)."""
    mp = import_moeplan()
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(meas))
    n_test = int(round(len(meas) * holdout))
    test = [meas[i] for i in order[:n_test]]
    train = [meas[i] for i in order[n_test:]]
    model = mp.train_forest(to_samples(train), hyper={"seed": seed})

    def errs(rows):
        if not rows:
            return []
        feats = np.array([[m.b, m.s, m.h] for m in rows], dtype=np.float64)
        pred = np.array([m.roofline_s for m in rows]) * model.predict_many(feats)
        meas_s = np.array([m.measured_s for m in rows])
        return list(np.abs(pred - meas_s) / meas_s)

    return model, errs(train), errs(test), test


def measured_cost_tensors(result, meas: List[Measurement]):
    """Per-module extension: the reference CostTensors (planner.py:82-132) with
    t_a / t_e replaced by the measured per-strategy times; t_c and c_switch
    are the reference's own (roofline comm at the measured NVLink bandwidth)."""
    mp = import_moeplan()
    t = result.tensors
    ta_p, ta_d = t.t_a_prefill.copy(), t.t_a_decode.copy()
    te_p, te_d = t.t_e_prefill.copy(), t.t_e_decode.copy()
    for m in meas:
        arr = {("attention", "prefill"): ta_p, ("attention", "decode"): ta_d,
               ("experts", "prefill"): te_p, ("experts", "decode"): te_d}[(m.module, m.stage)]
        arr[m.index] = m.measured_s
    return mp.CostTensors(t_a_prefill=ta_p, t_a_decode=ta_d, t_e_prefill=te_p, t_e_decode=te_d,
                          t_c_prefill=t.t_c_prefill, t_c_decode=t.t_c_decode, c_switch=t.c_switch)


# ------------------------------------------------------------ collectives --
def measure_collectives(volumes_bytes=(1 << 16, 1 << 20, 1 << 24, 1 << 27), reps: int = 10):
    """rho samples (communication CalibrationSamples) for AllReduce / AllGather /
    ReduceScatter / All-to-All over the WORLD group; run under torchrun on
    >= 2 GPUs.  Returns [(kind, logical_bytes, wire_bytes, seconds)]."""
    import torch.distributed as dist

    mp = import_moeplan()
    from moeplan.strategies import Collective, wire_bytes

    n = dist.get_world_size()
    out = []
    for vol in volumes_bytes:
        elems = vol // 2
        x = torch.randn(elems, device="cuda").to(BF16)
        for kind in ("allreduce", "allgather", "reducescatter", "all_to_all"):
            if kind == "allreduce":
                fn = lambda: dist.all_reduce(x)  # noqa: E731
                col = Collective("allreduce", vol, n, "expert")
            elif kind == "allgather":
                o = torch.empty(elems, device="cuda", dtype=BF16)
                fn = lambda: dist.all_gather_into_tensor(o, x[:elems // n])  # noqa: E731
                col = Collective("allgather", vol, n, "boundary")
            elif kind == "reducescatter":
                o = torch.empty(elems // n, device="cuda", dtype=BF16)
                fn = lambda: dist.reduce_scatter_tensor(o, x)  # noqa: E731
                col = Collective("allgather", vol, n, "boundary")
            else:
                o = torch.empty_like(x)
                fn = lambda: dist.all_to_all_single(o, x)  # noqa: E731
                col = Collective("all_to_all", vol * n, n, "expert")
            dist.barrier()
            t = _events_time(fn, reps)
            tt = torch.tensor([t], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            out.append((kind, float(vol), float(wire_bytes(col)), float(tt.item())))
    return out
