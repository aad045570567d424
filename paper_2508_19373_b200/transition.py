"""Stage-switch machinery of HAP's Eq.6 (reference
transition.py:1-267): the INT4 quantized-backup path measured on B200.

* ``Int4Backup`` keeps a GQI4 tensor (the reference's own container,
  quant.py:19-22, 119-154) in pinned host memory and restores it on device:
  asynchronous H2D upload of codes/scales/zero points, then the
  ``hap_int4_dequant`` kernel (bit-exact vs quant.py:dequantize in fp64, or
  bf16 weights).
* ``measure_dequant_table`` / ``measure_h2d_bandwidth`` produce the planner's
  inputs from measurements: a reference ``DequantTimeTable`` (transition.py:
  46-124; CSV ``n_gpus,v_dequant,seconds``) and ``host_to_device_bw`` for
  ``HardwareProfile`` (arch.py:80-101), replacing the synthetic 20e9
  params/s table (transition.py:36, 84-97).
"""

from __future__ import annotations

import statistics
from typing import Dict, Tuple

import torch

from . import ops as K
from .config import import_moeplan


class Int4Backup:
    """A GQI4 tensor resident in pinned host memory."""

    def __init__(self, q):
        self.group_size = int(q.group_size)
        self.n = int(q.original_len)
        self.codes = torch.from_numpy(q.codes.copy()).pin_memory()
        self.scales = torch.from_numpy(q.scales.copy()).pin_memory()
        self.zeros = torch.from_numpy(q.zero_points.copy()).pin_memory()

    @classmethod
    def from_values(cls, values, group_size: int = 128) -> "Int4Backup":
        mp = import_moeplan()
        return cls(mp.quantize_int4(values, group_size))

    def nbytes(self) -> int:
        return self.codes.numel() + 8 * (self.scales.numel() + self.zeros.numel())

    def restore(self, out: torch.Tensor, stream: torch.cuda.Stream = None) -> torch.Tensor:
        """Upload + dequantize into ``out`` (float64 or bf16, >= n elements) on ``stream``."""
        dev = out.device
        stream = stream or torch.cuda.current_stream(dev)
        with torch.cuda.stream(stream):
            codes = torch.empty(((self.codes.numel() + 3) // 4) * 4, dtype=torch.uint8, device=dev)
            codes[:self.codes.numel()].copy_(self.codes, non_blocking=True)
            scales = self.scales.to(dev, non_blocking=True)
            zeros = self.zeros.to(dev, non_blocking=True)
            K.int4_dequant(codes, scales, zeros, self.group_size, self.n, out)
        return out


# ------------------------------------------------------------------ reshard --
def _owned(lay, n_slices: int):
    """(unit, slice) pairs a rank holds — the reference's _ownership (transition.py:127-150):
    routed units [0, E), shared units E + u, each cut into n_slices TP slices."""
    per = lay.inter // n_slices
    i0, i1 = lay.inter_slice
    slices = range(i0 // per, i1 // per)
    e0, e1 = lay.experts
    own = {(e, s) for e in range(e0, e1) for s in slices}
    own |= {(lay.n_experts + u, s) for u in range(lay.n_shared) for s in slices}
    return own


def _unpack(cfg, w):
    """Packed RankWeights -> per-unit (gate [I_l,h], up [I_l,h], down^T [I_l,h]) views."""
    El, Il, h = w.n_experts_local, w.inter_local, cfg.hidden
    g13 = w.w13.view(El, Il // w.hw, 2, w.hw, h)
    gate = g13[:, :, 0].reshape(El, Il, h)
    up = g13[:, :, 1].reshape(El, Il, h)
    down_t = w.w2.transpose(1, 2)  # [El, Il, h]
    units = [(gate[e], up[e], down_t[e]) for e in range(El)]
    if cfg.n_shared:
        sil = w.shared_inter_local
        s13 = w.ws13.view(sil // w.hw_s, 2, w.hw_s, h)
        sg = s13[:, 0].reshape(sil, h)
        su = s13[:, 1].reshape(sil, h)
        sd = w.ws2.t()
        units += [(sg[u * Il:(u + 1) * Il], su[u * Il:(u + 1) * Il], sd[u * Il:(u + 1) * Il])
                  for u in range(cfg.n_shared)]
    return units


def _unit_views(cfg, w):
    """Per-unit (w13-like [.., 2I, h] interleaved tensor, row offset of the unit
    inside it, hw, w2-like [h, I_unit] view) for the routed experts then the
    shared units, without copying."""
    El, Il = w.n_experts_local, w.inter_local
    out = [(w.w13[e], 0, w.hw, w.w2[e]) for e in range(El)]
    if cfg.n_shared:
        out += [(w.ws13, u * Il, w.hw_s, w.ws2[:, u * Il:(u + 1) * Il]) for u in range(cfg.n_shared)]
    return out


def _gu_rows(t13, hw, r0, n, part):
    """Rows [r0, r0+n) of the gate (part 0) or up (part 1) half of an
    interleaved [2I, h] tensor as a strided [n/hw, hw, h] view (None when the
    rows do not align with the hw blocks)."""
    if r0 % hw or n % hw:
        return None
    v = t13.view(t13.shape[0] // (2 * hw), 2, hw, t13.shape[-1])
    return v[r0 // hw:(r0 + n) // hw, part]


def reshard_plan(lay_src_list, lay_dst_list, n_slices: int):
    """Deterministic transfer plan: for every destination rank, each (unit,
    slice) it needs and does not hold is fetched from one holder under the
    source layout (greedy: the holder with the least assigned volume)."""
    n = len(lay_src_list)
    own_src = [_owned(l, n_slices) for l in lay_src_list]
    own_dst = [_owned(l, n_slices) for l in lay_dst_list]
    sends = [[[] for _ in range(n)] for _ in range(n)]  # sends[src][dst] -> [(unit, slice)]
    load = [0] * n
    for r in range(n):
        for key in sorted(own_dst[r] - own_src[r]):
            holders = [q for q in range(n) if key in own_src[q]]
            q = min(holders, key=lambda x: (load[x], (x - r) % n))
            sends[q][r].append(key)
            load[q] += 1
    return own_src, own_dst, sends


def reshard_expert_weights(cfg, w, lay_src, lay_dst, group=None):
    """Move this rank's expert weights from layout lay_src to lay_dst with one
    all-to-all that carries exactly the (unit, slice) pieces each rank is
    missing (the per-device volume the reference charges in reshard_volume,
    transition.py:153-177).  Attention weights are unchanged (a plan has one
    attention strategy).  Returns a new RankWeights packed for lay_dst.

    Three phases (timed separately by scripts/measure_reshard.py): pack the
    pieces other ranks need (reshard_pack), one all_to_all_single, and
    re-pack the destination layout from local + received pieces
    (reshard_unpack)."""
    import torch.distributed as dist

    send, in_splits, out_splits, ctx = reshard_pack(cfg, w, lay_src, lay_dst)
    recv = torch.empty(sum(out_splits), dtype=send.dtype, device=send.device)
    if lay_src.n > 1:
        if recv.is_cuda and dist.get_backend(group) == "gloo":
            # single-GPU validation (ranks sharing one device): gloo stages through host memory
            rh = torch.empty(recv.shape, dtype=recv.dtype)
            dist.all_to_all_single(rh, send.cpu(), output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=group)
            recv.copy_(rh)
        else:
            dist.all_to_all_single(recv, send, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=group)
    return reshard_unpack(ctx, recv)


def _piece_views(buf, per: int, h: int):
    """A (unit, slice) piece on the wire: gate rows [per, h], up rows [per, h],
    then the down projection's columns as stored in w2, [h, per] (so both
    reshard phases copy row blocks and nothing is transposed)."""
    n = per * h
    return buf[:n].view(per, h), buf[n:2 * n].view(per, h), buf[2 * n:3 * n].view(h, per)


def _run_copies(pairs, bases=None, plan_key=None) -> None:
    """All the copies of one reshard phase: ONE hap_copy2d_batched launch for
    device tensors; host tensors (the CPU gloo tests of the host logic) copy
    pair by pair.  With ``bases`` / ``plan_key`` the launch's records are also
    kept relative to the phase's base tensors, so the next layer with the same
    layout pair replays them (``_replay``) without rebuilding any view."""
    if not pairs:
        if plan_key is not None:
            _COPY_PLANS[plan_key] = _np_empty_rel()
        return
    if pairs[0][0].is_cuda:
        from . import ops

        recs = ops.view_records(pairs)
        ops.copy_records(recs)
        if plan_key is not None:
            rel = _relativize(recs, bases)
            if rel is not None:
                _COPY_PLANS[plan_key] = rel
    else:
        for src, dst in pairs:
            dst.copy_(src)


# ------------------------------------------------- compiled reshard phases --
# The reshard plan and its copy records depend only on (model dims, source
# layout, destination layout, rank, packed weight shapes) — the same for every
# layer of a stage switch.  The first layer builds them from tensor views; the
# others replay the records with their own base pointers (one numpy add + one
# launch per phase).
_COPY_PLANS: dict = {}
_STATIC_PLANS: dict = {}


def _np_empty_rel():
    import numpy as np

    return np.zeros((0, 8), dtype=np.int64)


def _spans(bases):
    out = []
    for t in bases:
        if t is None:
            out.append((0, 0))
        else:
            p = t.data_ptr()
            out.append((p, p + t.numel() * t.element_size()))
    return out


def _relativize(recs, bases):
    """records [n, 6] -> [n, 8] (src base index, src offset, dst base index,
    dst offset, rows, row_bytes, src_pitch, dst_pitch), or None when a record
    lies outside every base (a temporary of the generic path: not replayable)."""
    import numpy as np

    spans = _spans(bases)

    def find(ptr):
        for i, (lo, hi) in enumerate(spans):
            if lo <= ptr < hi:
                return i, ptr - lo
        return None

    rel = np.empty((len(recs), 8), dtype=np.int64)
    for i, (sp_, dp_, rows, rb, ps, pd) in enumerate(recs.tolist()):
        fs, fd = find(sp_), find(dp_)
        if fs is None or fd is None:
            return None
        rel[i] = (fs[0], fs[1], fd[0], fd[1], rows, rb, ps, pd)
    return rel


def _replay(rel, bases) -> None:
    import numpy as np

    from . import ops

    if len(rel) == 0:
        return
    ptr = np.array([0 if t is None else t.data_ptr() for t in bases], dtype=np.int64)
    recs = np.empty((len(rel), 6), dtype=np.int64)
    recs[:, 0] = ptr[rel[:, 0]] + rel[:, 1]
    recs[:, 1] = ptr[rel[:, 2]] + rel[:, 3]
    recs[:, 2:] = rel[:, 4:]
    ops.copy_records(recs)


def _weights_key(w):
    ts = tuple(None if t is None else (tuple(t.shape), tuple(t.stride()), str(t.dtype))
               for t in (w.w13, w.w2, w.ws13, w.ws2))
    return ts + (w.hw, w.hw_s, w.n_experts_local, w.inter_local, w.shared_inter_local)


def _phase_key(cfg, w, lay_src, lay_dst):
    return (cfg.hidden, cfg.inter, cfg.n_experts, cfg.n_shared, cfg.n_q_heads, cfg.n_kv_heads,
            lay_src.deg, lay_src.rank, lay_dst.deg, str(w.w13.device), _weights_key(w))


def _static_plan(cfg, lay_src, lay_dst):
    """The host half of a reshard (who sends which (unit, slice) to whom), cached per layout pair."""
    from math import gcd

    from .layout import RankLayout

    key = (cfg.hidden, cfg.inter, cfg.n_experts, cfg.n_shared, cfg.n_q_heads, cfg.n_kv_heads,
           lay_src.deg, lay_src.rank, lay_dst.deg)
    hit = _STATIC_PLANS.get(key)
    if hit is not None:
        return hit
    n = lay_src.n
    tp_i, tp_j = lay_src.deg.e_tp, lay_dst.deg.e_tp
    n_slices = tp_i * tp_j // gcd(tp_i, tp_j)
    per = cfg.inter // n_slices
    h = cfg.hidden
    mk = lambda deg, r: RankLayout(deg, r, cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.inter, cfg.n_shared)  # noqa: E731
    srcs = [mk(lay_src.deg, r) for r in range(n)]
    dsts = [mk(lay_dst.deg, r) for r in range(n)]
    own_src, own_dst, sends = reshard_plan(srcs, dsts, n_slices)
    me = lay_src.rank
    piece_elems = 3 * per * h
    st = dict(n=n, per=per, h=h, own_src=own_src, sends=sends, me=me, e0=lay_src.experts[0],
              e1=lay_src.experts[1], s0=lay_src.inter_slice[0] // per, piece_elems=piece_elems,
              order=[(uu, s) for r in range(n) for (uu, s) in sends[me][r]],
              in_splits=[len(sends[me][r]) * piece_elems for r in range(n)],
              out_splits=[len(sends[q][me]) * piece_elems for q in range(n)])
    _STATIC_PLANS[key] = st
    return st


def reshard_pack(cfg, w, lay_src, lay_dst):
    """Phase 1 of the reshard: the send buffer (pieces this rank ships, grouped by
    destination) and the all-to-all splits; ctx carries what reshard_unpack needs."""
    st = _static_plan(cfg, lay_src, lay_dst)
    per, h, s0, e0, piece_elems, order = st["per"], st["h"], st["s0"], st["e0"], st["piece_elems"], st["order"]
    unpacked = []  # per-unit contiguous (gate, up, down^T), built only if a piece misses the fast path

    def unit_index(unit):
        return unit - e0 if unit < cfg.n_experts else (st["e1"] - e0) + (unit - cfg.n_experts)

    def local_piece(unit, s):
        """(gate [per,h], up [per,h], down [h,per]) views of a piece this rank holds."""
        if not unpacked:
            unpacked.append(_unpack(cfg, w))
        k = s - s0
        g, up, dt = (t[k * per:(k + 1) * per] for t in unpacked[0][unit_index(unit)])
        return g, up, dt.t()

    dev, dt = w.w13.device, w.w13.dtype
    send = torch.empty(len(order) * piece_elems, dtype=dt, device=dev)
    src_views = _unit_views(cfg, w)
    key = ("pack",) + _phase_key(cfg, w, lay_src, lay_dst)
    bases = [w.w13, w.w2, w.ws13, w.ws2, send]
    rel = _COPY_PLANS.get(key) if send.is_cuda else None
    if rel is not None:
        _replay(rel, bases)
    else:
        pairs = []
        for i, (uu, sl) in enumerate(order):
            # each piece is written once, straight from the packed source layout
            pg, pu, pd = _piece_views(send[i * piece_elems:(i + 1) * piece_elems], per, h)
            t13, base, hw_u, t2 = src_views[unit_index(uu)]
            r0 = base + (sl - s0) * per
            g, u_ = _gu_rows(t13, hw_u, r0, per, 0), _gu_rows(t13, hw_u, r0, per, 1)
            if g is None:
                lg, lu, ld = local_piece(uu, sl)
                pairs += [(lg, pg), (lu, pu), (ld, pd)]
            else:
                pairs += [(g, pg.view(per // hw_u, hw_u, h)), (u_, pu.view(per // hw_u, hw_u, h)),
                          (t2[:, (sl - s0) * per:(sl - s0 + 1) * per], pd)]
        _run_copies(pairs, bases, key if send.is_cuda else None)
    ctx = dict(cfg=cfg, w=w, lay_src=lay_src, lay_dst=lay_dst, n=st["n"], me=st["me"], per=per, h=h,
               own_src=st["own_src"], sends=st["sends"], local_piece=local_piece, piece_elems=piece_elems,
               src_views=src_views, unit_index=unit_index, s0=s0)
    return send, list(st["in_splits"]), list(st["out_splits"]), ctx


def reshard_unpack(ctx, recv):
    """Phase 3 of the reshard: the destination layout's RankWeights from this
    rank's own pieces plus the received buffer."""
    import dataclasses

    from .weights import interleave_gate_up, swiglu_half_width

    cfg, w, n, me, per = ctx["cfg"], ctx["w"], ctx["n"], ctx["me"], ctx["per"]
    own_src, sends, local_piece, piece_elems, h = (ctx["own_src"], ctx["sends"], ctx["local_piece"],
                                                  ctx["piece_elems"], ctx["h"])
    d = ctx["lay_dst"]
    de0, de1 = d.experts
    ds0, ds1 = d.inter_slice[0] // per, d.inter_slice[1] // per
    il = (ds1 - ds0) * per
    hw = swiglu_half_width(il)
    El_d = de1 - de0
    dev, dt = w.w13.device, w.w13.dtype
    units_d = list(range(de0, de1)) + [cfg.n_experts + u for u in range(cfg.n_shared)]
    sil = cfg.n_shared * il
    hw_s = swiglu_half_width(sil) if cfg.n_shared else 0
    # fast path: every destination slice lands on whole hw blocks of its tensor
    fast = per % hw == 0 and (not cfg.n_shared or (per % hw_s == 0 and il % hw_s == 0))
    if fast:
        w13 = torch.empty(El_d, 2 * il, h, dtype=dt, device=dev)
        w2 = torch.empty(El_d, h, il, dtype=dt, device=dev)
        ws13 = torch.empty(2 * sil, h, dtype=dt, device=dev) if cfg.n_shared else None
        ws2 = torch.empty(h, sil, dtype=dt, device=dev) if cfg.n_shared else None
        key = ("unpack",) + _phase_key(cfg, w, ctx["lay_src"], d)
        bases = [w.w13, w.w2, w.ws13, w.ws2, recv, w13, w2, ws13, ws2]
        rel = _COPY_PLANS.get(key) if recv.is_cuda else None
        if rel is not None:
            _replay(rel, bases)
        else:
            received = {}
            off = 0
            for q in range(n):
                for k_ in sends[q][me]:
                    received[k_] = _piece_views(recv[off:off + piece_elems], per, h)
                    off += piece_elems
            src_views, unit_index, s0 = ctx["src_views"], ctx["unit_index"], ctx["s0"]
            pairs = []
            for j, unit in enumerate(units_d):
                if unit < cfg.n_experts:
                    t13, base, hw_u, t2 = w13[j], 0, hw, w2[j]
                else:
                    u = unit - cfg.n_experts
                    t13, base, hw_u, t2 = ws13, u * il, hw_s, ws2[:, u * il:(u + 1) * il]
                for sl in range(ds0, ds1):
                    r0 = base + (sl - ds0) * per
                    gd, ud = _gu_rows(t13, hw_u, r0, per, 0), _gu_rows(t13, hw_u, r0, per, 1)
                    dcols = t2[:, (sl - ds0) * per:(sl - ds0 + 1) * per]
                    k_ = (unit, sl)
                    if k_ in own_src[me]:  # straight from this rank's own packed weights
                        st13, sbase, shw, st2 = src_views[unit_index(unit)]
                        sr0 = sbase + (sl - s0) * per
                        sg, su = _gu_rows(st13, shw, sr0, per, 0), _gu_rows(st13, shw, sr0, per, 1)
                        if sg is not None:
                            pairs += [(sg, gd), (su, ud), (st2[:, (sl - s0) * per:(sl - s0 + 1) * per], dcols)]
                            continue
                    pg, pu, pd = local_piece(*k_) if k_ in own_src[me] else received[k_]
                    pairs += [(pg.view(per // hw_u, hw_u, h), gd), (pu.view(per // hw_u, hw_u, h), ud), (pd, dcols)]
            _run_copies(pairs, bases, key if recv.is_cuda else None)
        return dataclasses.replace(w, w13=w13, w2=w2, hw=hw, ws13=ws13, ws2=ws2, hw_s=hw_s,
                                   n_experts_local=El_d, inter_local=il, shared_inter_local=sil)

    received = {}
    off = 0
    for q in range(n):
        for k_ in sends[q][me]:
            received[k_] = _piece_views(recv[off:off + piece_elems], per, h)
            off += piece_elems

    def piece(key):
        return local_piece(*key) if key in own_src[me] else received[key]

    def assemble(unit):
        ps = [piece((unit, s)) for s in range(ds0, ds1)]
        return (torch.cat([p[0] for p in ps]), torch.cat([p[1] for p in ps]),  # [il, h]
                torch.cat([p[2] for p in ps], dim=1))                          # [h, il]

    rout = [assemble(e) for e in range(de0, de1)]
    w13 = interleave_gate_up(torch.stack([g for g, _, _ in rout]), torch.stack([u for _, u, _ in rout]), hw)
    w2 = torch.stack([dn for _, _, dn in rout]).contiguous()
    ws13 = ws2 = None
    hw_s, sil = 0, 0
    if cfg.n_shared:
        sh = [assemble(cfg.n_experts + u) for u in range(cfg.n_shared)]
        sg = torch.cat([g for g, _, _ in sh])
        su = torch.cat([u for _, u, _ in sh])
        sil = sg.shape[0]
        hw_s = swiglu_half_width(sil)
        ws13 = interleave_gate_up(sg, su, hw_s)
        ws2 = torch.cat([dn for _, _, dn in sh], dim=1).contiguous()
    return dataclasses.replace(w, w13=w13, w2=w2, hw=hw, ws13=ws13, ws2=ws2, hw_s=hw_s,
                               n_experts_local=de1 - de0, inter_local=il, shared_inter_local=sil)


def _time(fn, reps: int = 5) -> float:
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


def measure_dequant_seconds(log2_sizes=range(10, 32), group_size: int = 128) -> Dict[int, float]:
    """Device seconds to dequantize 2^k parameters into bf16 (one B200)."""
    out: Dict[int, float] = {}
    max_n = 1 << max(log2_sizes)
    codes = torch.randint(0, 256, ((max_n + 1) // 2,), dtype=torch.uint8, device="cuda")
    n_groups = (max_n + group_size - 1) // group_size
    scales = torch.rand(n_groups, dtype=torch.float64, device="cuda") * 1e-2
    zeros = torch.randn(n_groups, dtype=torch.float64, device="cuda") * 1e-2
    dst = torch.empty(max_n, dtype=torch.bfloat16, device="cuda")
    for lg in log2_sizes:
        n = 1 << lg
        out[n] = _time(lambda: K.int4_dequant(codes, scales, zeros, group_size, n, dst))
    del codes, scales, zeros, dst
    torch.cuda.empty_cache()
    return out


def dequant_table(measured: Dict[int, float], max_gpus: int = 16, max_log2: int = 40):
    """Reference DequantTimeTable from per-device measurements.  Each device
    dequantizes its own shard concurrently, so every n_gpus row is the
    single-device curve; buckets beyond the largest measured size are
    extrapolated at the measured asymptotic rate (largest bucket)."""
    mp = import_moeplan()
    sizes = sorted(measured)
    top = sizes[-1]
    rate = top / measured[top]
    entries: Dict[Tuple[int, int], float] = {}
    n = 1
    while n <= max_gpus:
        for lg in range(10, max_log2 + 1):
            b = 1 << lg
            entries[(n, b)] = measured[b] if b in measured else max(measured[top], b / rate)
        n *= 2
    # enforce monotone rows (the reference table contract)
    for n2 in {k[0] for k in entries}:
        prev = 0.0
        for lg in range(10, max_log2 + 1):
            key = (n2, 1 << lg)
            entries[key] = max(entries[key], prev)
            prev = entries[key]
    return mp.DequantTimeTable(entries=entries)


def measure_h2d_bandwidth(nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Pinned host -> device copy bandwidth (bytes/s)."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    t = _time(lambda: dst.copy_(src, non_blocking=True), reps)
    return nbytes / t
