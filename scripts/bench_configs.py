"""Every BASELINE.json config measured on one B200 (the N=1 share of configs 2-5).

python scripts/bench_configs.py [out.json]

For each workload: one decoder block (random-init bf16 weights of the preset's
architecture, x ~ N(0, 1)) run through HapMoEBlock on the single-device plan,
CUDA-event time per step after warm-up (prefill: eager forwards; decode: graph
replays), and the fraction of roofline against the measured peaks in
MEASURED_PEAKS.json: prefill = the reference's algorithmic FLOPs
(attention_flops + expert_flops, arch.py:145-178, causal score/value term
halved) / dense bf16 peak; decode = algorithmic HBM bytes (experts touched,
attention weights, KV cache, router) / copy bandwidth.  Multi-GPU plans of
configs 3 and 5 are not measurable on a one-GPU box; the
Qwen2-57B decode sweep (config 4) runs B = 1..512 and records the decode plan
the reference ILP re-selects for 8 GPUs beside each row.
"""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_19373_b200.config import get_config, import_moeplan  # noqa: E402
from paper_2508_19373_b200.executor import HapMoEBlock, KVCache  # noqa: E402
from paper_2508_19373_b200.layout import PlanDegrees  # noqa: E402

mpl = import_moeplan()


def peaks():
    """MEASURED_PEAKS.json when the driver wrote one on this box, else bench.py's stated fallback."""
    from bench import load_peaks

    p = load_peaks()
    return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"]


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / steps)
    return statistics.median(ts)


def prefill(name, B, S, hbm, bf16, bf16s):
    cfg = get_config(name)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(B * S, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    ms = timed(lambda: blk.forward(x, "prefill", B, S), steps=5, warmup=3)
    spec = cfg.to_model_spec()
    T = B * S
    fl = mpl.attention_flops(spec, T, S) - 2 * T * S * cfg.hidden + mpl.expert_flops(spec, T)
    del blk
    torch.cuda.empty_cache()
    return {"workload": f"{name} block prefill {B}x{S}", "ms_per_step": ms, "tokens_per_s": T / ms * 1e3,
            "algorithmic_tflop": fl / 1e12, "achieved_tflops": fl / ms / 1e9, "frac_of_bf16_peak": fl / ms / 1e9 / bf16,
            "frac_of_sustained_bf16_peak": fl / ms / 1e9 / bf16s}


def decode(name, B, kv, hbm, bf16, bf16s):
    cfg = get_config(name)
    blk = HapMoEBlock(cfg, PlanDegrees(1, 1, 1, 1), None)
    cache = KVCache.empty(B, cfg.n_kv_heads, kv, cfg.head_dim, "cuda", random=True)
    pos = torch.full((B,), kv - 1, device="cuda", dtype=torch.int32)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(B, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    graph, _ = blk.capture_graph(x, "decode", B, kv_cache=cache, positions=pos)
    ms = timed(graph.replay, steps=100, warmup=20)
    touched = int(torch.unique(blk.last_routing[0]).numel())
    h, I, kvd = cfg.hidden, cfg.inter, cfg.kv_dim
    qd = cfg.n_q_heads * cfg.head_dim
    by = (touched * 3 * h * I * 2 + cfg.n_shared * 3 * h * I * 2 + (h * (qd + 2 * kvd) + qd * h) * 2
          + B * kv * 2 * kvd * 2 + (cfg.n_experts + (1 if cfg.n_shared else 0)) * h * 2)
    del graph, blk
    torch.cuda.empty_cache()
    return {"workload": f"{name} block decode B={B} kv={kv}", "ms_per_step": ms, "tokens_per_s": B / ms * 1e3,
            "experts_touched": touched, "algorithmic_gb": by / 1e9, "achieved_gbs": by / ms / 1e6,
            "frac_of_hbm_peak": by / ms / 1e6 / hbm}


def main():
    hbm, bf16, bf16s = peaks()
    rows = [
        prefill("mixtral-8x7b", 8, 2048, hbm, bf16, bf16s),
        decode("mixtral-8x7b", 64, 2048, hbm, bf16, bf16s),
        prefill("qwen1.5-moe-a2.7b", 8, 2048, hbm, bf16, bf16s),
        prefill("mixtral-8x22b", 16, 4096, hbm, bf16, bf16s),
    ]
    # config 4: the Qwen2-57B decode batch sweep 1-512; beside each row the
    # decode plan the reference ILP re-selects for 8 B200s (roofline tables)
    from paper_2508_19373_b200.plan import plan_for, stage_plan

    qcfg = get_config("qwen2-57b-a14b")
    for B in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512):
        row = decode("qwen2-57b-a14b", B, 2048, hbm, bf16, bf16s)
        sp = stage_plan(plan_for(qcfg, 8, B, 2048, 1), "decode")
        row["plan_n8_roofline"] = (f"attn(tp={sp.attention.tp_degree},dp={sp.attention.dp_degree})"
                                   f"+exp(tp={sp.expert.tp_degree},ep={sp.expert.ep_degree})")
        rows.append(row)
    out = {"device": torch.cuda.get_device_name(0),
           "peaks": {"hbm_gbs": hbm, "bf16_tflops": bf16, "bf16_tflops_sustained": bf16s},
           "plan": "single device: attn(tp=1,dp=1)+exp(tp=1,ep=1)", "data": "synthetic, random-init bf16 weights",
           "rows": rows}
    text = json.dumps(out, indent=1)
    print(text)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(text)


if __name__ == "__main__":
    main()
