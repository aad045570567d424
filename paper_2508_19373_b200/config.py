"""Block configuration: the reference's ``ModelSpec`` plus the HF-level details
the executor needs, and the B200 ``HardwareProfile``.

``ModelSpec`` (moeplan arch.py:16-77) fixes the dimensions the planner
reasons about; it leaves implicit what an executor must know to run the
block (router renormalisation, qkv bias, RMSNorm eps, RoPE theta).  These are
family-level facts of the HF models the presets describe (Mixtral: renorm,
no bias, eps 1e-5; Qwen2-MoE: no renorm, qkv bias, eps 1e-6, sigmoid-gated
shared expert) and are attached here without changing ModelSpec.
"""

from __future__ import annotations

import importlib
import os
import sys
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Dict

REPO = Path(__file__).resolve().parent.parent


def import_moeplan():
    """Import the reference planner (moeplan) — the upward API this executor plugs into.

    Looked up on sys.path first, then in ``baseline/_ref`` (the offline
    install of /root/reference that travels with the repo to the GPU box).
    """
    try:
        return importlib.import_module("moeplan")
    except ImportError:
        ref = os.environ.get("HAP_MOEPLAN_PATH", str(REPO / "baseline" / "_ref"))
        if ref not in sys.path:
            sys.path.append(ref)
        return importlib.import_module("moeplan")


@dataclass(frozen=True)
class BlockConfig:
    name: str
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    hidden: int
    n_experts: int
    n_shared: int          # shared units of `inter` (ModelSpec.n_shared_experts, arch.py:18-24)
    top_k: int
    inter: int             # ModelSpec.expert_inter_dim
    norm_topk_prob: bool = True
    qkv_bias: bool = False
    rope_theta: float = 1e6
    rms_eps: float = 1e-5
    dtype_bytes: int = 2

    def __post_init__(self):
        if self.n_q_heads * self.head_dim != self.hidden:
            raise ValueError("n_q_heads * head_dim must equal hidden (arch.py:57-61)")
        if self.n_q_heads % self.n_kv_heads:
            raise ValueError("n_kv_heads must divide n_q_heads (arch.py:62-65)")
        if self.top_k > self.n_experts:
            raise ValueError("top_k exceeds n_experts (arch.py:66-67)")

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def shared_inter(self) -> int:
        return self.n_shared * self.inter

    @property
    def family(self) -> str:
        return "qwen" if self.name.startswith("qwen") else "mixtral"

    def to_model_spec(self):
        mp = import_moeplan()
        return mp.ModelSpec(name=self.name, n_layers=self.n_layers, n_q_heads=self.n_q_heads,
                            n_kv_heads=self.n_kv_heads, head_dim=self.head_dim, hidden_dim=self.hidden,
                            n_experts=self.n_experts, n_shared_experts=self.n_shared, top_k=self.top_k,
                            expert_inter_dim=self.inter, dtype_bytes=self.dtype_bytes)

    @classmethod
    def from_model_spec(cls, spec) -> "BlockConfig":
        """Attach family defaults (by preset name) to a moeplan ModelSpec."""
        qwen = spec.name.startswith("qwen")
        return cls(name=spec.name, n_layers=spec.n_layers, n_q_heads=spec.n_q_heads, n_kv_heads=spec.n_kv_heads,
                   head_dim=spec.head_dim, hidden=spec.hidden_dim, n_experts=spec.n_experts,
                   n_shared=spec.n_shared_experts, top_k=spec.top_k, inter=spec.expert_inter_dim,
                   norm_topk_prob=not qwen, qkv_bias=qwen, rope_theta=1e6, rms_eps=1e-6 if qwen else 1e-5,
                   dtype_bytes=spec.dtype_bytes)


# The five BASELINE.json configs.  Mixtral-8x7B / Qwen presets mirror
# moeplan/presets/* (mixtral-8x7b:3-14, qwen1.5-moe-a2.7b:1-15,
# qwen2-57b-a14b:1-15); Mixtral-8x22B and the tiny config have no preset in
# the reference (SURVEY.md §0, §7 hard part 7): dimensions from the public
# model card / the BASELINE tiny description, with the tiny config's
# unspecified expert_inter_dim and n_kv_heads fixed to 1792 and 2.
PRESETS: Dict[str, BlockConfig] = {
    "tiny": BlockConfig(name="tiny", n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=64, hidden=512,
                        n_experts=8, n_shared=0, top_k=2, inter=1792),
    "mixtral-8x7b": BlockConfig(name="mixtral-8x7b", n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128,
                                hidden=4096, n_experts=8, n_shared=0, top_k=2, inter=14336),
    "mixtral-8x22b": BlockConfig(name="mixtral-8x22b", n_layers=56, n_q_heads=48, n_kv_heads=8, head_dim=128,
                                 hidden=6144, n_experts=8, n_shared=0, top_k=2, inter=16384),
    "qwen1.5-moe-a2.7b": BlockConfig(name="qwen1.5-moe-a2.7b", n_layers=24, n_q_heads=16, n_kv_heads=16,
                                     head_dim=128, hidden=2048, n_experts=60, n_shared=4, top_k=4, inter=1408,
                                     norm_topk_prob=False, qkv_bias=True, rms_eps=1e-6),
    "qwen2-57b-a14b": BlockConfig(name="qwen2-57b-a14b", n_layers=28, n_q_heads=28, n_kv_heads=4,
                                  head_dim=128, hidden=3584, n_experts=64, n_shared=8, top_k=8, inter=2560,
                                  norm_topk_prob=False, qkv_bias=True, rms_eps=1e-6),
}


def get_config(name: str) -> BlockConfig:
    try:
        return PRESETS[name]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; known: {sorted(PRESETS)}") from None


def scaled(cfg: BlockConfig, **kw) -> BlockConfig:
    return replace(cfg, **kw)


# Measured on this pool's B200s (MEASURED_PEAKS.json: bf16 1652.5 TF/s burst);
# NVLink: the pool's measured 8-rank all-reduce bus bandwidth, 725 GB/s at 1 GiB
# (B200_PROFILING.md; this run's boxes have one GPU, so it is not re-measured
# here); H2D: pinned host->device copy measured by scripts/measure_transition.py
# (profiles/r01_transition_measurements.json: 55.2 GB/s).
B200_PEAK_FLOPS = 1.6525e15
B200_HBM_BYTES = 180e9
B200_NVLINK_BW = 725e9
B200_H2D_BW = 55.2e9


def b200_hardware(n_devices: int, peak_flops: float = B200_PEAK_FLOPS, intra_node_bw: float = B200_NVLINK_BW,
                  host_to_device_bw: float = B200_H2D_BW):
    """moeplan HardwareProfile (arch.py:80-101) for an N x B200 NVSwitch node."""
    mp = import_moeplan()
    return mp.HardwareProfile(n_devices=n_devices, peak_flops=peak_flops, device_mem_bytes=B200_HBM_BYTES,
                              intra_node_bw=intra_node_bw, host_to_device_bw=host_to_device_bw,
                              link_label="nvlink5")
