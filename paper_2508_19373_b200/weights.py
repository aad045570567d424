"""Synthetic block weights and their per-rank packing for the kernels.

Canonical (unsharded) tensors use nn.Linear layouts and the names of the
oracle: wq/wk/wv [H*d, h], wo [h, Hq*d], router [E, h], w1/w3 [E, I, h]
(gate/up), w2 [E, h, I], shared ws1/ws3 [Is, h], ws2 [h, Is], wsg [1, h],
optional bq/bk/bv, ln1/ln2.  Every tensor is drawn from its own seeded
generator (seed = base_seed ^ crc32(name)), N(0, std^2) then rounded to bf16,
so every rank and every plan sees identical weights.

Packed per-rank layouts (HBM, all bf16, contiguous):
  wqkv   [(Hq_l + 2*Hkv_l) * d, h]    local q | k | v heads, one GEMM
  bqkv   [(Hq_l + 2*Hkv_l) * d]
  wo     [h, Hq_l * d]
  router [E (+1), h]                  row E = shared-expert gate when present
  w13    [E_l, 2*I_l, h]              gate/up interleaved in blocks of hw
                                      (hap_swiglu_half_width(I_l)) so one GEMM
                                      tile holds matching gate and up columns
  w2     [E_l, h, I_l]
  ws13   [2*Is_l, h], ws2 [h, Is_l]   shared expert, same interleave
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass
from typing import Dict, Optional

import torch

from .config import BlockConfig
from .layout import RankLayout


def weight_shapes(cfg: BlockConfig) -> Dict[str, tuple]:
    h, d = cfg.hidden, cfg.head_dim
    shapes = {
        "wq": (cfg.n_q_heads * d, h),
        "wk": (cfg.kv_dim, h),
        "wv": (cfg.kv_dim, h),
        "wo": (h, cfg.n_q_heads * d),
        "router": (cfg.n_experts, h),
        "w1": (cfg.n_experts, cfg.inter, h),
        "w3": (cfg.n_experts, cfg.inter, h),
        "w2": (cfg.n_experts, h, cfg.inter),
    }
    if cfg.qkv_bias:
        shapes.update({"bq": (cfg.n_q_heads * d,), "bk": (cfg.kv_dim,), "bv": (cfg.kv_dim,)})
    if cfg.n_shared:
        si = cfg.shared_inter
        shapes.update({"ws1": (si, h), "ws3": (si, h), "ws2": (h, si), "wsg": (1, h)})
    return shapes


def synthetic_weights(cfg: BlockConfig, device, seed: int = 0, std: float = 0.02,
                      names: Optional[list] = None) -> Dict[str, torch.Tensor]:
    """Full unsharded bf16 weights, deterministic per (seed, name, device type)."""
    out = {}
    for name, shape in weight_shapes(cfg).items():
        if names is not None and name not in names:
            continue
        g = torch.Generator(device=device)
        g.manual_seed((seed * 1_000_003) ^ zlib.crc32(name.encode()))
        t = torch.empty(shape, device=device, dtype=torch.float32)
        t.normal_(0.0, std, generator=g)
        out[name] = t.to(torch.bfloat16)
    for name in ("ln1", "ln2"):
        if names is not None and name not in names:
            continue
        g = torch.Generator(device=device)
        g.manual_seed((seed * 1_000_003) ^ zlib.crc32(name.encode()))
        t = torch.empty(cfg.hidden, device=device, dtype=torch.float32)
        t.normal_(0.0, 0.05, generator=g)
        out[name] = (1.0 + t).to(torch.bfloat16)
    return out


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor, hw: int) -> torch.Tensor:
    """[.., I, h] x 2 -> [.., 2I, h] with blocks [gate hw rows | up hw rows]."""
    *lead, I, h = gate.shape
    g = gate.reshape(*lead, I // hw, hw, h)
    u = up.reshape(*lead, I // hw, hw, h)
    return torch.stack([g, u], dim=-3).reshape(*lead, 2 * I, h).contiguous()


def swiglu_half_width(inter: int) -> int:
    """Same rule as hap_swiglu_half_width (gemm.cu): largest multiple of 8 <= 128 dividing inter."""
    for hw in range(128, 7, -8):
        if inter % hw == 0:
            return hw
    raise ValueError(f"no SwiGLU tile width divides inter={inter}")


@dataclass
class RankWeights:
    wqkv: torch.Tensor
    bqkv: Optional[torch.Tensor]
    wo: torch.Tensor
    ln1: torch.Tensor
    ln2: torch.Tensor
    router: torch.Tensor
    w13: torch.Tensor
    w2: torch.Tensor
    hw: int
    ws13: Optional[torch.Tensor]
    ws2: Optional[torch.Tensor]
    hw_s: int
    n_q_local: int
    n_kv_local: int
    n_experts_local: int
    inter_local: int
    shared_inter_local: int


def pack_rank_weights(cfg: BlockConfig, full: Dict[str, torch.Tensor], lay: RankLayout) -> RankWeights:
    d = cfg.head_dim
    q0, q1 = lay.q_heads
    k0, k1 = lay.kv_heads
    wqkv = torch.cat([full["wq"][q0 * d:q1 * d], full["wk"][k0 * d:k1 * d], full["wv"][k0 * d:k1 * d]], 0)
    bqkv = None
    if cfg.qkv_bias:
        bqkv = torch.cat([full["bq"][q0 * d:q1 * d], full["bk"][k0 * d:k1 * d], full["bv"][k0 * d:k1 * d]]).contiguous()
    wo = full["wo"][:, q0 * d:q1 * d].contiguous()
    router = full["router"]
    if cfg.n_shared:
        router = torch.cat([router, full["wsg"]], 0)
    e0, e1 = lay.experts
    i0, i1 = lay.inter_slice
    il = i1 - i0
    hw = swiglu_half_width(il)
    w13 = interleave_gate_up(full["w1"][e0:e1, i0:i1], full["w3"][e0:e1, i0:i1], hw)
    w2 = full["w2"][e0:e1, :, i0:i1].contiguous()
    ws13 = ws2 = None
    hw_s = 0
    sil = 0
    if cfg.n_shared:
        rows = torch.cat([torch.arange(a, b) for a, b in lay.shared_rows()]).to(full["ws1"].device)
        sil = rows.numel()
        hw_s = swiglu_half_width(sil)
        ws13 = interleave_gate_up(full["ws1"][rows], full["ws3"][rows], hw_s)
        ws2 = full["ws2"][:, rows].contiguous()
    return RankWeights(wqkv=wqkv.contiguous(), bqkv=bqkv, wo=wo, ln1=full["ln1"].contiguous(),
                       ln2=full["ln2"].contiguous(), router=router.contiguous(), w13=w13, w2=w2, hw=hw,
                       ws13=ws13, ws2=ws2, hw_s=hw_s, n_q_local=q1 - q0, n_kv_local=k1 - k0,
                       n_experts_local=e1 - e0, inter_local=il, shared_inter_local=sil)
