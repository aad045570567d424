"""Generate golden vectors for the oracle from HF transformers (5.5.0, fp32, CPU).

The reference package (moeplan) has no forward implementation, so the
op semantics of the MoE block are pinned against the HF decoder layers its
presets describe: MixtralDecoderLayer (mixtral-8x7b preset) and
Qwen2MoeDecoderLayer (qwen1.5-moe / qwen2-57b presets).  Weights come from
``oracle.moe_block.random_weights`` (numpy PCG64, deterministic across
machines), so fixtures only store inputs and outputs.

Run from the repo root:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.moe_block import BlockSpec, random_weights  # noqa: E402

OUT = Path(__file__).resolve().parent

CASES = {
    # Mixtral-style: GQA, no bias, renormalised top-2, no shared experts.
    "mixtral_small": (BlockSpec(hidden=256, n_q_heads=4, n_kv_heads=2, head_dim=64, n_experts=8, top_k=2,
                                inter=384, n_shared=0, norm_topk_prob=True, qkv_bias=False,
                                rope_theta=1e6, rms_eps=1e-5), 2, 24),
    # Qwen2-MoE-style: qkv bias, 4 shared units, no renorm, top-4 of 16.
    "qwen2moe_small": (BlockSpec(hidden=256, n_q_heads=4, n_kv_heads=4, head_dim=64, n_experts=16, top_k=4,
                                 inter=128, n_shared=4, norm_topk_prob=False, qkv_bias=True,
                                 rope_theta=1e6, rms_eps=1e-6), 2, 20),
}


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))


def hf_layer(name: str, spec: BlockSpec, W):
    if name.startswith("mixtral"):
        from transformers import MixtralConfig
        from transformers.models.mixtral.modeling_mixtral import MixtralDecoderLayer, MixtralRotaryEmbedding

        cfg = MixtralConfig(hidden_size=spec.hidden, intermediate_size=spec.inter,
                            num_attention_heads=spec.n_q_heads, num_key_value_heads=spec.n_kv_heads,
                            head_dim=spec.head_dim, num_local_experts=spec.n_experts,
                            num_experts_per_tok=spec.top_k, rms_norm_eps=spec.rms_eps,
                            rope_theta=spec.rope_theta, max_position_embeddings=4096)
        cfg._attn_implementation = "eager"
        layer = MixtralDecoderLayer(cfg, 0)
        rot = MixtralRotaryEmbedding(cfg)
        moe = layer.mlp
        moe.gate.weight.data = _t(W["router"])
        moe.experts.gate_up_proj.data = torch.cat([_t(W["w1"]), _t(W["w3"])], dim=1)
        moe.experts.down_proj.data = _t(W["w2"])
    else:
        from transformers import Qwen2MoeConfig
        from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeDecoderLayer, Qwen2MoeRotaryEmbedding

        cfg = Qwen2MoeConfig(hidden_size=spec.hidden, moe_intermediate_size=spec.inter,
                             shared_expert_intermediate_size=spec.shared_inter,
                             num_attention_heads=spec.n_q_heads, num_key_value_heads=spec.n_kv_heads,
                             num_experts=spec.n_experts, num_experts_per_tok=spec.top_k,
                             norm_topk_prob=spec.norm_topk_prob, rms_norm_eps=spec.rms_eps,
                             rope_theta=spec.rope_theta, max_position_embeddings=4096, qkv_bias=True,
                             decoder_sparse_step=1, mlp_only_layers=[])
        cfg._attn_implementation = "eager"
        layer = Qwen2MoeDecoderLayer(cfg, 0)
        rot = Qwen2MoeRotaryEmbedding(cfg)
        moe = layer.mlp
        moe.gate.weight.data = _t(W["router"])
        moe.experts.gate_up_proj.data = torch.cat([_t(W["w1"]), _t(W["w3"])], dim=1)
        moe.experts.down_proj.data = _t(W["w2"])
        moe.shared_expert.gate_proj.weight.data = _t(W["ws1"])
        moe.shared_expert.up_proj.weight.data = _t(W["ws3"])
        moe.shared_expert.down_proj.weight.data = _t(W["ws2"])
        moe.shared_expert_gate.weight.data = _t(W["wsg"])
        layer.self_attn.q_proj.bias.data = _t(W["bq"])
        layer.self_attn.k_proj.bias.data = _t(W["bk"])
        layer.self_attn.v_proj.bias.data = _t(W["bv"])
    at = layer.self_attn
    at.q_proj.weight.data = _t(W["wq"])
    at.k_proj.weight.data = _t(W["wk"])
    at.v_proj.weight.data = _t(W["wv"])
    at.o_proj.weight.data = _t(W["wo"])
    layer.input_layernorm.weight.data = _t(W["ln1"])
    layer.post_attention_layernorm.weight.data = _t(W["ln2"])
    return layer.eval(), rot


def run_case(name: str):
    spec, n_seqs, S = CASES[name]
    W = random_weights(spec, seed=1234, bf16=True)
    rng = np.random.default_rng(99)
    x = rng.standard_normal((n_seqs, S, spec.hidden)).astype(np.float32)
    layer, rot = hf_layer(name, spec, W)
    xt = torch.from_numpy(x)
    pos = torch.arange(S).unsqueeze(0).expand(n_seqs, S)
    cos, sin = rot(xt, pos)
    mask = torch.full((S, S), float("-inf")).triu(1)[None, None].expand(n_seqs, 1, S, S)
    with torch.no_grad():
        out = layer(xt, position_embeddings=(cos, sin), attention_mask=mask, position_ids=pos)
        if isinstance(out, tuple):
            out = out[0]
        # router probabilities on the post-attention normalised input
        res = xt + layer.self_attn(layer.input_layernorm(xt), position_embeddings=(cos, sin),
                                   attention_mask=mask)[0]
        hn = layer.post_attention_layernorm(res).reshape(-1, spec.hidden)
        probs, top_w, top_i = layer.mlp.gate(hn)
    np.savez_compressed(OUT / f"{name}.npz", x=x, out=out.numpy(), h1=res.numpy(), hn=hn.numpy(),
                        probs=probs.numpy(), topk_idx=top_i.numpy().astype(np.int32),
                        topk_w=top_w.float().numpy())
    print(f"{name}: wrote {OUT / (name + '.npz')}")


if __name__ == "__main__":
    torch.manual_seed(0)
    for n in CASES:
        run_case(n)
