"""Full-model loop: n_layers HAP blocks of one plan, prefill that fills the
per-layer KV caches, then decode steps that append to them.

This turns block tokens/s into the end-to-end latency the reference's
simulator predicts (simulate.py:78-114: prefill = n_layers * (attn + experts
+ comm); decode = output_len * n_layers * (...)), so the predicted-vs-measured
comparison covers the whole model (scripts/e2e_model.py).  Weights are random
per layer (seed + layer), generated and packed one layer at a time.

A plan whose expert layout differs between prefill and decode switches
between the stages with switch_to_decode(): every layer's expert weights are
resharded by one minimal-volume all-to-all (transition.reshard_expert_weights,
the volume the reference charges in transition.py:153-177).
"""

from __future__ import annotations

from typing import List, Optional

import torch

from .config import BlockConfig
from .executor import HapMoEBlock, KVCache, PagedKV, PagedKVCache
from .layout import PlanDegrees, replica_sequences
from .weights import synthetic_weights


class HapModel:
    def __init__(self, cfg: BlockConfig, attention, expert, *, n_layers: Optional[int] = None, rank: int = 0,
                 device=None, seed: int = 0, ops=None, comm=None):
        self.cfg = cfg
        self.n_layers = n_layers or cfg.n_layers
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.blocks: List[HapMoEBlock] = []
        for layer in range(self.n_layers):
            W = synthetic_weights(cfg, self.device, seed=seed * 1000 + layer)
            blk = HapMoEBlock(cfg, attention, expert, rank=rank, device=self.device, weights=W, ops=ops,
                              comm=comm if comm is not None else (self.blocks[0].comm if self.blocks else None))
            del W
            self.blocks.append(blk)
            if self.device.type == "cuda":
                torch.cuda.empty_cache()
        self.deg = self.blocks[0].deg
        self.lay = self.blocks[0].lay

    @classmethod
    def from_plan(cls, cfg: BlockConfig, plan, **kw) -> "HapModel":
        """Model laid out for the plan's prefill stage; call switch_to_decode()
        before decoding when the plan's expert layouts differ (Eq.6)."""
        m = cls(cfg, plan.attention, plan.expert_prefill, **kw)
        m._attention, m._expert_decode = plan.attention, plan.expert_decode
        return m

    def switch_expert_layout(self, expert) -> float:
        """HAP's stage switch: reshard every layer's expert weights to a new
        expert strategy with one minimal-volume all-to-all per layer
        (transition.reshard_expert_weights); returns the device seconds spent
        (max over ranks when distributed)."""
        from .transition import reshard_expert_weights

        new_deg = PlanDegrees(self.deg.a_tp, self.deg.a_dp, expert.tp_degree, expert.ep_degree,
                              getattr(expert, "dp_degree", 1))
        if new_deg == self.deg:
            return 0.0
        lay_dst = None
        cuda = self.device.type == "cuda"
        if cuda:
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
        new_blocks, comm = [], None
        for blk in self.blocks:
            from .layout import RankLayout

            lay_dst = RankLayout(new_deg, blk.lay.rank, self.cfg.n_q_heads, self.cfg.n_kv_heads, self.cfg.n_experts,
                                 self.cfg.inter, self.cfg.n_shared)
            w_new = reshard_expert_weights(self.cfg, blk.w, blk.lay, lay_dst)
            nb = HapMoEBlock.from_rank_weights(self.cfg, new_deg, blk.lay.rank, w_new, device=self.device,
                                               ops=blk.ops, comm=comm)
            comm = nb.comm
            new_blocks.append(nb)
        seconds = 0.0
        if cuda:
            e.record()
            torch.cuda.synchronize()
            seconds = s.elapsed_time(e) / 1e3
        if cuda:
            torch.cuda.synchronize()
        for blk in self.blocks:  # release the old layout's peer mappings / symmetric buffers
            blk.close()
        self.blocks, self.deg, self.lay = new_blocks, new_deg, new_blocks[0].lay
        return seconds

    def switch_to_decode(self) -> float:
        exp = getattr(self, "_expert_decode", None)
        return 0.0 if exp is None else self.switch_expert_layout(exp)

    def new_caches(self, batch: int, max_len: int, paged: bool = False, page: int = 64,
                   n_pages: Optional[int] = None) -> List[KVCache]:
        """Per-layer KV caches for this rank's sequences: contiguous
        [B_l, Hkv_l, max_len, d], or (paged) views of one PagedKV whose pages
        are allocated as the sequences grow (prefill / decode_step call
        ``ensure``)."""
        s0, s1 = replica_sequences(batch, self.deg.a_dp, self.lay.a_rep)
        nkv = self.blocks[0].w.n_kv_local
        if paged:
            state = PagedKV(self.n_layers, max(s1 - s0, 1), nkv, self.cfg.head_dim, max_len, self.device, page=page,
                            n_pages=n_pages)
            return [state.layer(i) for i in range(self.n_layers)]
        return [KVCache.empty(max(s1 - s0, 1), nkv, max_len, self.cfg.head_dim, self.device)
                for _ in range(self.n_layers)]

    def prefill(self, x_local: torch.Tensor, batch: int, seq_len: int, caches: List[KVCache]) -> torch.Tensor:
        h = x_local
        if caches and isinstance(caches[0], PagedKVCache):
            caches[0].state.ensure(seq_len)
        for blk, cache in zip(self.blocks, caches):
            h = blk.forward(h, "prefill", batch, seq_len, kv_cache=cache)
        return h

    def decode_step(self, x_local: torch.Tensor, batch: int, caches: List[KVCache],
                    positions: torch.Tensor, max_position: Optional[int] = None) -> torch.Tensor:
        """One decode step through every layer.  ``max_position`` (the caller's
        host-side bound on ``positions``) is checked against the caches once,
        without reading the device tensor back."""
        h = x_local
        if max_position is None and positions.is_cuda and not torch.cuda.is_current_stream_capturing() and caches:
            max_position = caches[0].check_positions(positions)  # one read-back for the whole step
        if caches and isinstance(caches[0], PagedKVCache) and max_position is not None:
            caches[0].state.ensure(max_position + 1)  # the new token's page
        for blk, cache in zip(self.blocks, caches):
            h = blk.forward(h, "decode", batch, kv_cache=cache, positions=positions, max_position=max_position)
        return h

    def capture_decode(self, x_static: torch.Tensor, batch: int, caches: List[KVCache], positions: torch.Tensor):
        """One CUDA graph for a whole decode step (all layers).  `positions` is
        read on device, so advancing it in place between replays is enough."""
        if self.deg.e_ep > 1 or self.lay.n > 1:
            raise RuntimeError("graph capture is supported for single-device, non-EP plans")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                self.decode_step(x_static, batch, caches, positions)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.decode_step(x_static, batch, caches, positions)
        return g, out
