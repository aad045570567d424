"""HAP MoE-block executor: runs one (AttentionStrategy, ExpertStrategy) plan
emitted by the reference planner (moeplan planner.py:527-549) on B200s.

Per rank and per call (prefill or decode) the block is

  attention module (heads sharded by attention tp, sequences by attention dp)
    rmsnorm -> QKV GEMM (+bias) -> RoPE -> attention core -> O GEMM (+residual)
    -> AllReduce over the attention-TP group                (strategies.py:314-322)
  boundary: all-gather of normalised tokens when the expert shard spans
    several attention replicas (DP -> TP, strategies.py:324-332)
  expert module (experts sharded by ep, intermediate dim by expert tp)
    router/top-k -> permute -> [EP: count exchange + dispatch All-to-All]
    -> grouped GEMM gate/up (+SwiGLU) -> grouped GEMM down
    -> [EP: combine All-to-All] -> weighted combine (+shared expert, +residual)
  reduce-scatter over the expert-TP group (TP -> DP, strategies.py:324-342),
  then all-gather over the attention-TP group back to the input layout.

Every compute op is a libhap_kernels launch (``CudaOps``); the executor never
computes on the host and has no fallback.  A different ``ops`` object can be
injected only by the test-suite's CPU multi-process tests, which exercise the
collective schedule on gloo (see tests/test_executor_dist.py).
"""

from __future__ import annotations

import os
from contextlib import contextmanager
from dataclasses import dataclass
from typing import Optional

import torch

from . import ops as K
from .comm import Comm
from .config import BlockConfig
from .layout import PlanDegrees, RankLayout, replica_sequences, tokens_per_replica
from .weights import RankWeights, pack_rank_weights, synthetic_weights

BF16 = torch.bfloat16
_SHARED_SIDE_STREAM_MAX_T = 512  # decode-size batches: shared expert on a side stream


def _shared_sm_budget(device) -> int:
    """SMs the side-stream shared expert may use (half; HAP_SHARED_SMS overrides, 0 = all)."""
    env = os.environ.get("HAP_SHARED_SMS")
    if env is not None:
        return int(env)
    return torch.cuda.get_device_properties(device).multi_processor_count // 2


def _maybe_peer_allreduce(comm) -> None:
    """HAP_PEER_AR=1 / HAP_NVLS_AR=1: decode-size all-reduces of this block's
    groups go through the one-shot peer-memory kernel or the NVLS in-switch
    reduction (both graph capturable); opt-in until measured on a multi-GPU box."""

    if comm is None or comm.lay.n == 1:
        return
    if os.environ.get("HAP_NVLS_AR", "0") == "1":  # in-switch reduction (NVSwitch multicast)
        comm.enable_peer_allreduce(["attn_tp_group", "exp_tp_group"], mode="nvls")
    elif os.environ.get("HAP_PEER_AR", "0") == "1":
        comm.enable_peer_allreduce(["attn_tp_group", "exp_tp_group"])


def _boundary_peer_default() -> bool:
    """DP<->TP boundary pushed through peer memory (HAP_BOUNDARY_PEER=1) instead of
    NCCL AllGather + ReduceScatter; opt-in until measured on a multi-GPU box."""

    return os.environ.get("HAP_BOUNDARY_PEER", "0") == "1"


def _ep_peer_default() -> bool:
    """EP dispatch/combine through peer-mapped buffers (HAP_EP_PEER=1) instead of
    NCCL all-to-alls; opt-in until measured on a multi-GPU box."""

    return os.environ.get("HAP_EP_PEER", "0") == "1"


# HAP_FUSED_NORM=1: decode runs the attention norm inside the QKV launch
# (hap_rmsnorm_gemm_qkv_rope).  Off by default: one launch fewer and 1.7-3.6 us
# faster in isolation, but the graph-replayed decode step measured +15 us
# (Mixtral-8x7B B=1) / +1 us (Qwen2-57B B=1) with it (profiles/r02_fused_norm_ab.txt)
_FUSED_NORM = os.environ.get("HAP_FUSED_NORM", "0") == "1"


class CudaOps:
    """The product compute backend: every method launches a kernel of
    libhap_kernels.so through the C-ABI (ops.py).  Construction fails loudly
    if CUDA or the library is unavailable."""

    def __init__(self):
        from . import _lib

        if not torch.cuda.is_available():
            raise RuntimeError("HAP executor requires a CUDA device (sm_100a); there is no CPU path")
        _lib.load()

    rmsnorm = staticmethod(K.rmsnorm)
    gemm = staticmethod(K.gemm)
    gemm_qkv_rope = staticmethod(K.gemm_qkv_rope)
    rmsnorm_qkv_rope = staticmethod(K.rmsnorm_qkv_rope)
    grouped_gemm = staticmethod(K.grouped_gemm)
    rope_qk = staticmethod(K.rope_qk)
    attn_prefill = staticmethod(K.attn_prefill)
    attn_decode = staticmethod(K.attn_decode)
    kv_cache_fill = staticmethod(K.kv_cache_fill)
    kv_cache_fill_paged = staticmethod(K.kv_cache_fill_paged)
    attn_decode_paged = staticmethod(K.attn_decode_paged)
    router_topk = staticmethod(K.router_topk)
    moe_permute = staticmethod(K.moe_permute)
    moe_combine = staticmethod(K.moe_combine)
    grouped_gemm_scatter = staticmethod(K.grouped_gemm_scatter)
    peer_copy_rows = staticmethod(K.peer_copy_rows)
    rmsnorm_multi = staticmethod(K.rmsnorm_multi)
    moe_combine_chunked = staticmethod(K.moe_combine_chunked)
    reduce_slots = staticmethod(K.reduce_slots)
    peer_broadcast_i32 = staticmethod(K.peer_broadcast_i32)
    ep_exchange_plan = staticmethod(K.ep_exchange_plan)
    permute_workspace_bytes = staticmethod(K.permute_workspace_bytes)
    attn_decode_workspace_bytes = staticmethod(K.attn_decode_workspace_bytes)


@dataclass
class KVCache:
    """Head-major cache of this rank's local kv heads: [bpr, Hkv_l, max_len, d]."""

    k: torch.Tensor
    v: torch.Tensor

    @classmethod
    def empty(cls, bpr: int, n_kv_local: int, max_len: int, head_dim: int, device, random: bool = False):
        shape = (bpr, n_kv_local, max_len, head_dim)
        if random:
            k = torch.randn(shape, device=device, dtype=torch.float32).to(BF16)
            v = torch.randn(shape, device=device, dtype=torch.float32).to(BF16)
        else:
            k = torch.zeros(shape, device=device, dtype=BF16)
            v = torch.zeros(shape, device=device, dtype=BF16)
        return cls(k, v)

    @property
    def max_len(self) -> int:
        return int(self.k.shape[2])

    def check_positions(self, positions: torch.Tensor) -> int:
        """Raise ValueError unless every decode position is inside the cache
        (0 <= pos < max_len).  Reads device positions back (one sync), so the
        graph-captured decode path validates on the host side instead
        (HapModel.capture_decode callers own their position counter); the
        kernels themselves never write or read outside a sequence's rows."""
        if positions.numel() == 0:
            return 0
        lo, hi = int(positions.min()), int(positions.max())
        if lo < 0 or hi >= self.max_len:
            raise ValueError(f"decode positions [{lo}, {hi}] outside the KV cache (max_len {self.max_len})")
        return hi


class PagedKV:
    """Paged KV cache for a stack of layers (the full-model loop, SURVEY §8(f)
    row 3): per layer a pool of pages [n_pages, Hkv_l, page, d] for k and for v,
    and ONE int32 block table [B, max_pages] shared by every layer (a sequence's
    j-th page has the same id in every layer's pool).  Pages are handed out on
    the host as sequences grow (``ensure``) and returned by ``release``; the
    device table is refreshed by one small copy only when it changed, so a
    captured decode graph stays valid while the table rows it reads are updated
    in place."""

    def __init__(self, n_layers: int, batch: int, n_kv_local: int, head_dim: int, max_len: int, device,
                 page: int = 64, n_pages: Optional[int] = None):
        if page % 16:
            raise ValueError("page size must be a multiple of 16 (the decode kernel's key chunk)")
        self.page, self.batch = page, batch
        self.max_pages = -(-max_len // page)
        self.n_pages = n_pages if n_pages is not None else batch * self.max_pages
        shape = (self.n_pages, n_kv_local, page, head_dim)
        self.k = [torch.zeros(shape, device=device, dtype=BF16) for _ in range(n_layers)]
        self.v = [torch.zeros(shape, device=device, dtype=BF16) for _ in range(n_layers)]
        self.table_host = torch.full((batch, self.max_pages), -1, dtype=torch.int32)
        self.table = self.table_host.to(device)
        self.free = list(range(self.n_pages - 1, -1, -1))
        self.held = [0] * batch  # pages held per sequence

    @property
    def max_len(self) -> int:
        return self.max_pages * self.page

    def ensure(self, length: int, seqs=None) -> None:
        """Pages for keys [0, length) of every sequence in `seqs` (default: all)."""
        need = -(-length // self.page)
        if need > self.max_pages:
            raise ValueError(f"length {length} exceeds the paged cache (max_len {self.max_len})")
        changed = False
        for b in (range(self.batch) if seqs is None else seqs):
            while self.held[b] < need:
                if not self.free:
                    raise RuntimeError("paged KV cache out of pages")
                self.table_host[b, self.held[b]] = self.free.pop()
                self.held[b] += 1
                changed = True
        if changed:
            self.table.copy_(self.table_host, non_blocking=False)

    def release(self, b: int) -> None:
        """Return sequence b's pages to the pool (its rows become unallocated)."""
        self.free.extend(int(x) for x in self.table_host[b, :self.held[b]].tolist())
        self.table_host[b] = -1
        self.held[b] = 0
        self.table.copy_(self.table_host)

    def layer(self, i: int) -> "PagedKVCache":
        return PagedKVCache(self.k[i], self.v[i], self)


@dataclass
class PagedKVCache:
    """One layer's view of a PagedKV (what HapMoEBlock.forward takes as kv_cache)."""

    k: torch.Tensor
    v: torch.Tensor
    state: PagedKV

    @property
    def max_len(self) -> int:
        return self.state.max_len

    def check_positions(self, positions: torch.Tensor) -> int:
        return KVCache.check_positions(self, positions)


class HapMoEBlock:
    """One MoE decoder block laid out for one plan on one rank."""

    def __init__(self, cfg: BlockConfig, attention, expert, *, rank: int = 0, device=None, seed: int = 0,
                 weights: Optional[dict] = None, ops=None, comm: Optional[Comm] = None):
        self.cfg = cfg
        self.deg = attention if isinstance(attention, PlanDegrees) and expert is None else \
            PlanDegrees.from_strategies(attention, expert)
        self.lay = RankLayout(self.deg, rank, cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.inter,
                              cfg.n_shared)
        self.ops = ops if ops is not None else CudaOps()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        full = weights if weights is not None else synthetic_weights(cfg, self.device, seed)
        self.w: RankWeights = pack_rank_weights(cfg, full, self.lay)
        del full
        self.comm = comm if comm is not None else (Comm(self.lay) if self.lay.n > 1 else None)
        _maybe_peer_allreduce(self.comm)
        self.last_routing = None  # (topk_idx, dst_of_row, seg) of the last expert call, for parity tests
        self.capture = None       # set to {} to keep references to intermediates (tests only)
        self.timers = None        # set to {} to record CUDA events around each kernel phase (bench)
        self.ep_peer = _ep_peer_default()
        self.boundary_peer = _boundary_peer_default()

    @classmethod
    def from_rank_weights(cls, cfg: BlockConfig, deg: PlanDegrees, rank: int, w: RankWeights, *, device=None,
                          ops=None, comm: Optional[Comm] = None) -> "HapMoEBlock":
        """A block over already-packed weights (e.g. after an expert-layout switch)."""
        blk = cls.__new__(cls)
        blk.cfg, blk.deg = cfg, deg
        blk.lay = RankLayout(deg, rank, cfg.n_q_heads, cfg.n_kv_heads, cfg.n_experts, cfg.inter, cfg.n_shared)
        blk.ops = ops if ops is not None else CudaOps()
        blk.device = torch.device(device) if device is not None else w.w13.device
        blk.w = w
        blk.comm = comm if comm is not None else (Comm(blk.lay) if blk.lay.n > 1 else None)
        _maybe_peer_allreduce(blk.comm)
        blk.last_routing = None
        blk.capture = None
        blk.timers = None
        blk.ep_peer = _ep_peer_default()
        blk.boundary_peer = _boundary_peer_default()
        return blk

    @classmethod
    def from_plan(cls, cfg: BlockConfig, plan, stage: str = "prefill", **kw) -> "HapMoEBlock":
        """Build from a moeplan Plan (planner.py:142-166) for one stage."""
        exp = plan.expert_prefill if stage == "prefill" else plan.expert_decode
        return cls(cfg, plan.attention, exp, **kw)

    # ------------------------------------------------------------ helpers --
    @contextmanager
    def _timed(self, name):
        if self.timers is None:
            yield
            return
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        yield
        e.record()
        self.timers.setdefault(name, []).append((s, e))

    def _prefill_positions(self, bpr: int, S: int, rows: int) -> torch.Tensor:
        key = (bpr, S, rows)
        cache = getattr(self, "_pos_cache", None)
        if cache is None or cache[0] != key:
            pos = torch.zeros(rows, dtype=torch.int32)
            pos[:bpr * S] = torch.arange(S, dtype=torch.int32).repeat(bpr)
            self._pos_cache = (key, pos.to(self.device))
        return self._pos_cache[1]

    def _coll(self, name, *args):
        if self.comm is None:
            return None
        return getattr(self.comm, name)(*args)

    def _attn_rows(self, batch: int, seq: int):
        bpr, rows = tokens_per_replica(batch, self.deg.a_dp, seq, self.lay.n)
        s0, s1 = replica_sequences(batch, self.deg.a_dp, self.lay.a_rep)
        return bpr, rows, s1 - s0

    # ------------------------------------------------------------ forward --
    def forward(self, x_local: torch.Tensor, stage: str, batch: int, seq_len: int = 1,
                kv_cache: Optional[KVCache] = None, positions: Optional[torch.Tensor] = None,
                max_position: Optional[int] = None) -> torch.Tensor:
        """x_local: this attention replica's tokens [n_seqs_local * seq_len, h]
        (prefill) or [n_seqs_local, h] (decode); returns the block output in
        the same layout.  positions (decode): int32 [n_seqs_local] current
        lengths (the new token's position).  Positions are validated against
        the cache on the host: from ``max_position`` (the caller's own bound,
        no device read-back) when given, else from a host ``positions``
        tensor, else by reading the device tensor back (one sync; skipped
        under graph capture — the kernels never touch rows outside a
        sequence's cache either way)."""
        if stage == "prefill":
            return self._forward(x_local, batch, seq_len, decode=False, kv_cache=kv_cache)
        if stage == "decode":
            if kv_cache is None or positions is None:
                raise ValueError("decode needs a kv_cache and positions")
            return self._forward(x_local, batch, 1, decode=True, kv_cache=kv_cache, positions=positions,
                                 max_position=max_position)
        raise ValueError(f"unknown stage {stage!r}")

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor, batch: int, seq_len: int,
                     n_chunks: int = 1) -> torch.Tensor:
        """Prefill from/to pinned HOST buffers, asynchronous and pipelined.

        The call queues H2D (copy stream) -> block forward (current stream) ->
        D2H (second copy stream) and returns; device input buffers are double
        buffered across calls, so the H2D of call i+1 overlaps the forward of
        call i and the D2H of call i overlaps the forward of call i+1 (a
        serving loop streams batches this way).  ``out_host`` is valid after
        ``host_sync()`` + a stream synchronisation.  With n_chunks > 1 the batch
        is additionally split into sequence chunks inside the call (sequences
        are independent in the block, so the output equals one forward over the
        whole batch; single-device plans).  Under a multi-GPU plan, ``batch`` is
        the global batch and x_host this rank's replica rows, as for forward()."""
        if self.lay.n > 1 and n_chunks != 1:
            raise RuntimeError("sequence chunking is single-device; under a multi-GPU plan use n_chunks=1")
        if not (x_host.is_pinned() and out_host.is_pinned()):
            raise ValueError("host buffers must be pinned for asynchronous copies")
        n_chunks = max(1, min(n_chunks, batch))
        while batch % n_chunks:
            n_chunks -= 1
        # forward() takes the global batch; x_host holds this rank's replica rows
        bc = batch // n_chunks
        rows = x_host.shape[0] // n_chunks
        st = getattr(self, "_host", None)
        if st is None or st["rows"] != rows or st["n_chunks"] != n_chunks:
            st = {"rows": rows, "n_chunks": n_chunks, "i": 0,
                  "streams": (torch.cuda.Stream(), torch.cuda.Stream()),
                  "slots": [{"bufs": [torch.empty(rows, self.cfg.hidden, device=self.device, dtype=BF16)
                                      for _ in range(n_chunks)], "free": [None] * n_chunks} for _ in range(2)]}
            self._host = st
        h2d, d2h = st["streams"]
        slot = st["slots"][st["i"] % 2]
        st["i"] += 1
        comp = torch.cuda.current_stream()
        for c in range(n_chunks):
            buf = slot["bufs"][c]
            if slot["free"][c] is not None:  # the forward that last read this buffer has finished
                h2d.wait_event(slot["free"][c])
            else:
                h2d.wait_stream(comp)
            with torch.cuda.stream(h2d):
                buf.copy_(x_host[c * rows:(c + 1) * rows], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(h2d)
            comp.wait_event(loaded)
            o = self.forward(buf, "prefill", bc, seq_len)
            done = torch.cuda.Event()
            done.record(comp)
            slot["free"][c] = done
            d2h.wait_event(done)
            with torch.cuda.stream(d2h):
                out_host[c * rows:(c + 1) * rows].copy_(o, non_blocking=True)
                o.record_stream(d2h)
        return out_host

    def host_sync(self) -> None:
        """Order the current stream after every queued forward_host copy."""
        st = getattr(self, "_host", None)
        if st is not None:
            comp = torch.cuda.current_stream()
            for s in st["streams"]:
                comp.wait_stream(s)

    def capture_graph(self, x_static: torch.Tensor, stage: str, batch: int, seq_len: int = 1,
                kv_cache: Optional[KVCache] = None, positions: Optional[torch.Tensor] = None):
        """Capture one forward into a CUDA graph over static buffers; returns
        (graph, out_static).  Replaying the graph re-runs every kernel of the
        block with no host work (decode is launch-bound otherwise).  Only for
        plans without host synchronisation (no EP count exchange) on one GPU."""
        if not self.graph_capturable(batch, seq_len):
            raise RuntimeError("graph capture needs one device, a peer-memory boundary / EP plan, or a non-EP plan "
                               "whose all-reduces fit the one-shot peer all-reduce (HAP_PEER_AR=1)")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):  # warm-up: kernel attributes, allocator pools
                self.forward(x_static, stage, batch, seq_len, kv_cache=kv_cache, positions=positions)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.forward(x_static, stage, batch, seq_len, kv_cache=kv_cache, positions=positions)
        return g, out

    def _forward(self, x_local, batch, S, decode, kv_cache=None, positions=None, max_position=None):
        cfg, w, lay, ops = self.cfg, self.w, self.lay, self.ops
        dev = self.device
        h, d = cfg.hidden, cfg.head_dim
        bpr, rows, n_seq = self._attn_rows(batch, S)
        T_real = n_seq * S
        if x_local.shape != (T_real, h):
            raise ValueError(f"x_local must be [{T_real}, {h}] for this rank, got {tuple(x_local.shape)}")
        if rows != T_real:
            x = torch.zeros(rows, h, device=dev, dtype=BF16)
            x[:T_real].copy_(x_local)
        else:
            x = x_local.contiguous()

        # ---------------- attention module
        # decode, opt-in: the norm rides in the QKV launch (GEMV at 1-2 rows
        # stages the normalised rows itself; bit-identical to the two launches)
        fused_norm = decode and _FUSED_NORM and hasattr(ops, "rmsnorm_qkv_rope")
        if not fused_norm:
            with self._timed("norm"):
                xn = ops.rmsnorm(x, w.ln1, cfg.rms_eps)
        nq, nkv = w.n_q_local, w.n_kv_local
        if decode:
            if max_position is not None:  # the caller's host-side length: no device read-back
                if n_seq and not 0 <= max_position < kv_cache.max_len:
                    raise ValueError(f"decode position {max_position} outside the KV cache "
                                     f"(max_len {kv_cache.max_len})")
            elif not positions.is_cuda or not torch.cuda.is_current_stream_capturing():
                kv_cache.check_positions(positions[:n_seq])
            if not positions.is_cuda:
                positions = positions.to(dev, non_blocking=True)
            if rows == n_seq and positions.dtype == torch.int32 and positions.is_contiguous():
                pos = positions
            else:
                pos = torch.zeros(rows, device=dev, dtype=torch.int32)
                pos[:n_seq].copy_(positions)
        else:
            pos = self._prefill_positions(bpr, S, rows)
        # QKV projection with RoPE fused into the GEMM epilogue
        with self._timed("qkv"):
            if fused_norm:
                qkv = ops.rmsnorm_qkv_rope(x, w.ln1, cfg.rms_eps, w.wqkv, pos, nq + nkv, d, cfg.rope_theta,
                                           bias=w.bqkv)
            else:
                qkv = ops.gemm_qkv_rope(xn, w.wqkv, pos, nq + nkv, d, cfg.rope_theta, bias=w.bqkv)
        attn = torch.zeros(rows, nq * d, device=dev, dtype=BF16) if rows != T_real else \
            torch.empty(rows, nq * d, device=dev, dtype=BF16)
        paged = isinstance(kv_cache, PagedKVCache)
        if decode:
            ws = torch.empty(ops.attn_decode_workspace_bytes(max(n_seq, 1), nq, d, kv_cache.max_len),
                             device=dev, dtype=torch.uint8)
            if n_seq and paged:
                ops.attn_decode_paged(qkv[:n_seq], kv_cache.k, kv_cache.v, kv_cache.state.table[:n_seq],
                                      pos[:n_seq], nq, nkv, d, attn[:n_seq], ws)
            elif n_seq:
                ops.attn_decode(qkv[:n_seq], kv_cache.k[:n_seq], kv_cache.v[:n_seq], pos[:n_seq], nq, nkv, d,
                                attn[:n_seq], ws)
        elif n_seq:
            if paged:  # keep this prefill's k/v in the sequences' pages
                ops.kv_cache_fill_paged(qkv, nq, nkv, d, n_seq, S, kv_cache.k, kv_cache.v,
                                        kv_cache.state.table[:n_seq])
            elif kv_cache is not None:  # keep this prefill's k/v for the decode steps that follow
                ops.kv_cache_fill(qkv, nq, nkv, d, n_seq, S, kv_cache.k, kv_cache.v)
            with self._timed("attn"):
                ops.attn_prefill(qkv, nq, nkv, d, n_seq, S, attn)
        with self._timed("o_proj"):
            h1 = ops.gemm(attn, w.wo, residual=x if lay.a_tp_rank == 0 else None)
        c = rows // self.deg.a_tp  # rows this rank owns after the reduce-scatter
        # expert shard = this rank's 1/a_tp of its replica (expert tp 1): the
        # attention partial sums are reduce-scattered straight onto the shards
        # (RS here + the AllGather after the experts = the AllReduce the
        # reference charges, strategies.py:314-322), else all-reduced
        rs_attn = self.deg.a_tp > 1 and self.deg.e_tp == 1
        if rs_attn:
            h1c = torch.empty(c, h, device=dev, dtype=BF16)
            self.comm.reduce_scatter(h1c, h1, "attn_tp_group")
            h1 = h1c
        else:
            self._coll("all_reduce", h1, "attn_tp_group")
        S_e, a_dp = lay.n_shards, self.deg.a_dp
        pb = self._peer_boundary(rows) if self._uses_peer_boundary() else None
        if pb is not None:
            # boundary all-gather pushed by the norm into every rank's gather buffer
            with self._timed("norm"):
                ops.rmsnorm_multi(h1, w.ln2, cfg.rms_eps, pb.ag_tab, h)
            pb.barrier()
            hn = hn_s = pb.gath.local[:pb.n * rows]
        else:
            with self._timed("norm"):
                hn = ops.rmsnorm(h1, w.ln2, cfg.rms_eps)

        # ---------------- boundary: attention layout -> expert shard
        if pb is not None:
            pass
        elif rs_attn:
            hn_s = hn
        elif S_e < a_dp:
            R = a_dp // S_e
            hn_s = torch.empty(R * rows, h, device=dev, dtype=BF16)
            self.comm.all_gather(hn_s, hn, "gather_group")
        elif S_e > a_dp:
            P = S_e // a_dp
            p = lay.shard % P
            rs = rows // P
            hn_s = hn[p * rs:(p + 1) * rs]
        else:
            hn_s = hn
        if self.capture is not None:
            self.capture.update(qkv=qkv, attn=attn, h1=h1, hn=hn, hn_s=hn_s)

        # ---------------- expert module (partial over expert tp)
        residual = h1 if rs_attn else h1[lay.a_tp_rank * c:(lay.a_tp_rank + 1) * c]
        if pb is not None:
            # expert-TP reduce-scatter pushed by the combine, summed by the owner in rank order
            self._experts(hn_s, residual, res_row0=lay.e_tp_rank * c, res_rows=c, push=pb)
            pb.barrier()
            out = ops.reduce_slots(pb.slots.local, pb.n, rows, torch.empty(rows, h, device=dev, dtype=BF16))
            return out[:T_real]
        y = self._experts(hn_s, residual, res_row0=lay.e_tp_rank * c, res_rows=c)

        # ---------------- back to the attention layout
        if self._peer_allreduce_back(y):
            # pure TP: RS + AG over one group == one all-reduce, done one-shot over peer memory
            return self.comm.all_reduce(y, "attn_tp_group")[:T_real]
        if self.deg.e_tp > 1:
            chunk = torch.empty(c, h, device=dev, dtype=BF16)
            self.comm.reduce_scatter(chunk, y, "exp_tp_group")
        else:
            chunk = y
        if self.deg.a_tp > 1:
            out = torch.empty(rows, h, device=dev, dtype=BF16)
            self.comm.all_gather(out, chunk, "attn_tp_group")
        else:
            out = chunk
        return out[:T_real]

    def _side_stream(self):
        st = getattr(self, "_side", None)
        if st is None or st.device != self.device:
            st = self._side = torch.cuda.Stream(device=self.device)
        return st

    def _uses_peer_boundary(self) -> bool:
        """Peer-memory boundary: pure attention DP, and the expert shard gathers
        exactly the expert-TP group (gather group == expert-TP group)."""
        c = self.comm
        return (self.boundary_peer and c is not None and self.deg.a_tp == 1 and self.deg.e_ep == 1
                and self.lay.n_shards < self.deg.a_dp and self.deg.e_tp > 1
                and c.groups["gather_group"][0] == c.groups["exp_tp_group"][0])

    def _peer_boundary(self, rows: int):
        """Symmetric gather / slot buffers for `rows` rows per replica, (re)allocated
        collectively (every rank of the group sees the same rows)."""
        from .peer import PeerBoundary

        pb = getattr(self, "_pb", None)
        if pb is not None and pb.rows == rows:
            return pb
        if pb is not None:
            torch.cuda.synchronize()
            self.comm.barrier("exp_tp_group")
            pb.close()
        self._pb = PeerBoundary(rows, self.cfg.hidden, self.device, self.comm._g("exp_tp_group"),
                                self.comm.groups["exp_tp_group"][0])
        return self._pb

    def _peer_allreduce_back(self, y) -> bool:
        c = self.comm
        return (c is not None and self.deg.e_tp > 1 and self.deg.a_tp == self.deg.e_tp
                and c.groups["exp_tp_group"][0] == c.groups["attn_tp_group"][0]
                and c.uses_peer_allreduce("attn_tp_group") and c.peer_ar["attn_tp_group"].fits(y))

    def graph_capturable(self, batch: Optional[int] = None, seq_len: int = 1) -> bool:
        """True when a forward issues no host synchronisation and no NCCL call:
        one device; the DP<->TP boundary or attention-DP x EP over peer memory;
        or a non-EP plan whose collectives all run through the one-shot peer
        all-reduce (HAP_PEER_AR=1) — which needs the call's tensors to fit the
        all-reduce buffer, so that case is only claimed for a known ``batch``."""
        if self.lay.n == 1:
            return True
        if self._uses_peer_boundary():
            return True
        c = self.comm
        if (self.deg.e_ep > 1 and self.ep_peer and self.deg.a_tp == 1 and self.deg.e_tp == 1
                and self.lay.n_shards == self.deg.a_dp):
            return True  # attention DP x expert EP: every exchange is a peer store + device barrier
        if not (self.deg.e_ep == 1 and self.lay.n_shards == self.deg.a_dp and c is not None
                and c.size("gather_group") == 1):
            return False
        if batch is None:
            return False
        _, rows, _ = self._attn_rows(batch, seq_len)
        n_elems = rows * self.cfg.hidden
        for k in ("attn_tp_group", "exp_tp_group"):
            if c.size(k) > 1 and not (c.uses_peer_allreduce(k) and c.peer_ar[k].n_max >= n_elems):
                return False
        # the expert side must close with the one-shot all-reduce, not RS + AG over NCCL
        return self.deg.e_tp == 1 or (self.deg.a_tp == self.deg.e_tp
                                      and c.groups["exp_tp_group"][0] == c.groups["attn_tp_group"][0])

    def _experts(self, hn_s, residual, res_row0, res_rows, push=None):
        cfg, w, lay, ops = self.cfg, self.w, self.lay, self.ops
        dev = self.device
        T, h = hn_s.shape
        E, k = cfg.n_experts, cfg.top_k
        # shared expert (Qwen): independent of the routed path; on small (decode)
        # batches its weight-streaming GEMMs run on a side stream, concurrently
        # with router -> permute -> grouped GEMMs, so neither path's launch ramp
        # and tail idle the HBM (fork/join by events: CUDA-graph capturable).
        # They keep to half the SMs: unbounded, their persistent grids take every
        # SM and the routed path waits for them (Qwen2-57B decode B=1
        # 249 -> 226 us, B=2 316-348 -> 279-310 us, profiles/r02_shared_sms.txt)
        ys, side = None, None
        if cfg.n_shared:
            if hn_s.is_cuda and T <= _SHARED_SIDE_STREAM_MAX_T:
                side = self._side_stream()
                side.wait_stream(torch.cuda.current_stream())
                sms = _shared_sm_budget(hn_s.device)
                with torch.cuda.stream(side):
                    ys = ops.gemm(ops.gemm(hn_s, w.ws13, swiglu_half=w.hw_s, sm_budget=sms), w.ws2, sm_budget=sms)
            else:
                ys = ops.gemm(ops.gemm(hn_s, w.ws13, swiglu_half=w.hw_s), w.ws2)
        idx = torch.empty(T, k, device=dev, dtype=torch.int32)
        tw = torch.empty(T, k, device=dev, dtype=torch.float32)
        sg = torch.empty(T, device=dev, dtype=torch.float32) if cfg.n_shared else None
        with self._timed("router"):
            ops.router_topk(hn_s, w.router, E, k, cfg.norm_topk_prob, bool(cfg.n_shared), idx, tw, sg)
        R = T * k
        x_perm = torch.empty(R, h, device=dev, dtype=BF16)
        dst = torch.empty(R, device=dev, dtype=torch.int32)
        seg = torch.empty(E + 1, device=dev, dtype=torch.int32)
        ws = torch.empty(max(ops.permute_workspace_bytes(R, E), 16), device=dev, dtype=torch.uint8)
        with self._timed("permute"):
            ops.moe_permute(idx.view(-1), E, hn_s, k, x_perm, dst, seg, ws)
        self.last_routing = (idx, dst, seg)
        if self.capture is not None:
            self.capture.update(topk_w=tw, shared_gate=sg)
        il = w.inter_local
        if self.deg.e_ep == 1:
            H = torch.empty(R, il, device=dev, dtype=BF16)
            with self._timed("gate_up"):
                ops.grouped_gemm(x_perm, w.w13, E, seg, H, swiglu_half=w.hw)
            Y = torch.empty(R, h, device=dev, dtype=BF16)
            with self._timed("down"):
                ops.grouped_gemm(H, w.w2, E, seg, Y)
        elif self.ep_peer:
            Y = self._ep_experts_peer(x_perm, seg)
        else:
            Y = self._ep_experts(x_perm, seg)
        if side is not None:  # join the shared expert's stream before the combine reads ys
            main = torch.cuda.current_stream()
            main.wait_stream(side)
            ys.record_stream(main)
        if push is not None:  # chunk q of the partial sums straight into slot `me` of rank q
            with self._timed("combine"):
                ops.moe_combine_chunked(Y, dst, tw, T, k, h, push.rs_tab, push.rows, push.me, residual=residual,
                                        shared_y=ys, shared_gate=sg, res_row0=res_row0, res_rows=res_rows)
            return None
        out = torch.empty(T, h, device=dev, dtype=BF16)
        with self._timed("combine"):
            ops.moe_combine(Y, dst, tw, T, k, out, residual=residual, shared_y=ys, shared_gate=sg,
                            res_row0=res_row0, res_rows=res_rows)
        return out

    def _ep_experts(self, x_perm, seg):
        """EP dispatch -> local grouped GEMMs -> combine (strategies.py:334-340)."""
        w, ops, comm = self.w, self.ops, self.comm
        dev = self.device
        ep, El, h = self.deg.e_ep, w.n_experts_local, self.cfg.hidden
        counts = (seg[1:] - seg[:-1]).contiguous()           # [E] rows per global expert, dest-group major
        recv_counts = torch.empty_like(counts)                # [ep * El]: from src s, local expert j
        comm.all_to_all(recv_counts, counts, [El] * ep, [El] * ep, "a2a_group")
        both = torch.cat([counts, recv_counts]).cpu()         # the one host sync of the EP path
        send = both[:ep * El].view(ep, El).sum(1).tolist()
        rc = both[ep * El:].view(ep, El)
        recv = rc.sum(1).tolist()
        n_recv = int(sum(recv))
        x_recv = torch.empty(n_recv, h, device=dev, dtype=BF16)
        comm.all_to_all(x_recv, x_perm, recv, send, "a2a_group")
        # received rows are grouped (src rank, local expert): one GEMM segment each
        seg_r = torch.zeros(ep * El + 1, dtype=torch.int32)
        seg_r[1:] = torch.cumsum(rc.reshape(-1), 0)
        grp = torch.arange(El, dtype=torch.int32).repeat(ep)
        seg_r, grp = seg_r.to(dev, non_blocking=True), grp.to(dev, non_blocking=True)
        il = w.inter_local
        H = torch.empty(n_recv, il, device=dev, dtype=BF16)
        Y_r = torch.empty(n_recv, h, device=dev, dtype=BF16)
        if n_recv:
            with self._timed("gate_up"):
                ops.grouped_gemm(x_recv, w.w13, El, seg_r, H, swiglu_half=w.hw, seg_group=grp)
            with self._timed("down"):
                ops.grouped_gemm(H, w.w2, El, seg_r, Y_r, seg_group=grp)
        Y = torch.empty(x_perm.shape[0], h, device=dev, dtype=BF16)
        comm.all_to_all(Y, Y_r, send, recv, "a2a_group")
        return Y


    def close(self) -> None:
        """Release peer mappings (every rank, before a barrier and shutdown)."""
        for name in ("_pb", "_pe"):
            if getattr(self, name, None) is not None:
                getattr(self, name).close()
                setattr(self, name, None)
        for par in getattr(self.comm, "peer_ar", {}).values():
            par.close()

    # ------------------------------------------------ EP over peer memory --
    def _peer_ep(self, rows: int):
        """Worst-case-sized symmetric EP buffers for `rows` permuted rows per rank,
        grown collectively (every rank of the EP group has the same row count)."""
        from .peer import PeerEP

        pe = getattr(self, "_pe", None)
        if pe is not None and pe.rows >= rows:
            return pe
        if pe is not None:
            torch.cuda.synchronize()
            self.comm.barrier("a2a_group")
            pe.close()
        self._pe = PeerEP(rows, self.cfg.hidden, self.w.inter_local, self.cfg.n_experts, self.device,
                          self.comm._g("a2a_group"), self.comm.groups["a2a_group"][0])
        return self._pe

    def _ep_experts_peer(self, x_perm, seg):
        """EP dispatch -> local grouped GEMMs -> combine with both all-to-alls done
        as direct stores into peer-mapped buffers and the exchange planned on the
        device (peer.PeerEP): no count reaches the host.  Received rows sit in
        (source rank, local expert) blocks exactly as in _ep_experts, so the
        GEMMs see the same rows and the results are identical."""
        w, ops = self.w, self.ops
        R, h = x_perm.shape
        pe = self._peer_ep(R)
        E, El = self.cfg.n_experts, pe.El
        ops.peer_broadcast_i32(seg, pe.segs_tab, pe.me * (E + 1) * 4)
        pe.barrier()                                          # every rank's segment offsets have landed
        ops.ep_exchange_plan(pe.segs.local, pe.n, El, pe.me, pe.dst_row0, pe.seg_r, pe.seg_dst_row0)
        ops.peer_copy_rows(x_perm, seg, pe.dst_base, pe.dst_row0, h)
        pe.barrier()                                          # every rank's rows have landed
        with self._timed("gate_up"):
            ops.grouped_gemm(pe.recv.local, w.w13, El, pe.seg_r, pe.H, swiglu_half=w.hw, seg_group=pe.grp)
        with self._timed("down"):
            ops.grouped_gemm_scatter(pe.H, w.w2, El, pe.seg_r, pe.grp, pe.seg_dst, pe.seg_dst_row0, h)
        pe.barrier()                                          # every expert output is back at its source
        return pe.y.local[:R]


def forward(block: HapMoEBlock, hidden: torch.Tensor, stage: str, batch: int, seq_len: int = 1,
            kv_cache: Optional[KVCache] = None, positions: Optional[torch.Tensor] = None) -> torch.Tensor:
    """hap.forward: the block's plan applied to this rank's tokens."""
    return block.forward(hidden, stage, batch, seq_len, kv_cache=kv_cache, positions=positions)
