"""End-to-end Mixtral-8x7B (all 32 layers, random weights) on one B200:
prefill 8 x 2048 then 64 graph-replayed decode steps, measured, against the
reference simulator's prediction (simulate.py:78-114) with (a) its roofline
cost tensors and (b) B200-measured module tables for this exact scenario.

  python scripts/e2e_model.py [--layers 32] [--out gpurun_out/r01_e2e_model.json]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2508_19373_b200 import calib  # noqa: E402
from paper_2508_19373_b200.config import get_config, import_moeplan  # noqa: E402
from paper_2508_19373_b200.model import HapModel  # noqa: E402
from paper_2508_19373_b200.plan import plan_for  # noqa: E402

mp = import_moeplan()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--input-len", type=int, default=2048)
    ap.add_argument("--output-len", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/r02_e2e_model.json")
    ap.add_argument("--page", type=int, default=64, help="also run the decode steps over a paged KV cache")
    args = ap.parse_args()
    cfg = get_config(args.config)
    L = args.layers or cfg.n_layers
    B, S, O = args.batch, args.input_len, args.output_len

    res = plan_for(cfg, 1, B, S, O)
    p = res.plan
    t0 = time.time()
    model = HapModel.from_plan(cfg, p, n_layers=L)
    build_s = time.time() - t0

    x = torch.randn(B * S, cfg.hidden, device="cuda").to(torch.bfloat16)
    caches = model.new_caches(B, S + O)
    model.prefill(x, B, S, caches)  # warm-up (also fills caches)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    model.prefill(x, B, S, caches)
    ev[1].record()
    pos = torch.full((B,), S, device="cuda", dtype=torch.int32)
    xd = torch.randn(B, cfg.hidden, device="cuda").to(torch.bfloat16)
    graph, _ = model.capture_decode(xd, B, caches, pos)
    pos.fill_(S)
    torch.cuda.synchronize()
    ev[2].record()
    for _ in range(O):
        graph.replay()
        pos.add_(1)
    ev[3].record()
    torch.cuda.synchronize()
    prefill_s = ev[0].elapsed_time(ev[1]) / 1e3
    decode_s = ev[2].elapsed_time(ev[3]) / 1e3
    measured_total = prefill_s + decode_s

    # the same decode steps over a paged KV cache (pages handed out as the
    # sequences grow: one host-side ensure per step, a table copy at page edges)
    paged = None
    if args.page:
        pcaches = model.new_caches(B, S + O, paged=True, page=args.page)
        model.prefill(x, B, S, pcaches)
        st = pcaches[0].state
        st.ensure(S + 1)
        pos.fill_(S)
        pgraph, _ = model.capture_decode(xd, B, pcaches, pos)
        pos.fill_(S)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(O):
            st.ensure(S + i + 1)
            pgraph.replay()
            pos.add_(1)
        e1.record()
        torch.cuda.synchronize()
        pd = e0.elapsed_time(e1) / 1e3
        paged = {"page_tokens": args.page, "decode_s": pd, "decode_ms_per_token_step": pd / O * 1e3,
                 "pages_held": sum(st.held), "vs_contiguous": pd / decode_s}

    # predictions: reference simulate() on roofline tensors and on measured module tables
    spec = cfg.to_model_spec()
    scen = mp.InferenceScenario(B, S, O)
    roof = mp.simulate(p.indices(), res.tensors, spec, scen)
    meas = calib.measure_catalog(cfg, 1, B, S, O, reps=5)
    tens = calib.measured_cost_tensors(res, meas)
    cal = mp.simulate(p.indices(), tens, spec, scen)
    scale = L / cfg.n_layers  # simulate counts cfg.n_layers layers
    report = {
        "config": f"{cfg.name} x {L} layers, B={B}, input {S}, output {O}, 1 B200, plan {p.attention.label()}+"
                  f"{p.expert_prefill.label()}",
        "weights_build_s": build_s,
        "measured": {"prefill_s": prefill_s, "decode_s": decode_s, "decode_ms_per_token_step": decode_s / O * 1e3,
                     "total_s": measured_total, "prefill_tokens_per_s": B * S / prefill_s,
                     "decode_tokens_per_s": B * O / decode_s},
        "measured_paged_kv": paged,
        "predicted_roofline": {"prefill_s": roof.prefill_s * scale, "decode_s": roof.decode_s * scale,
                               "total_s": (roof.prefill_s + roof.decode_s) * scale},
        "predicted_measured_tables": {"prefill_s": cal.prefill_s * scale, "decode_s": cal.decode_s * scale,
                                      "total_s": (cal.prefill_s + cal.decode_s) * scale},
    }
    for k in ("predicted_roofline", "predicted_measured_tables"):
        report[k]["rel_err_total"] = abs(report[k]["total_s"] - measured_total) / measured_total
        report[k]["rel_err_prefill"] = abs(report[k]["prefill_s"] - prefill_s) / prefill_s
        report[k]["rel_err_decode"] = abs(report[k]["decode_s"] - decode_s) / decode_s
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(report, indent=1))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
