"""Time the two local phases of the prefill->decode expert reshard on one B200
at full Mixtral-8x7B size (one layer), for the N=8 layout switches the planner
can emit: pack (the pieces rank r ships) and unpack (re-pack the destination
layout from its own + received pieces).  The all-to-all in between moves the
reference's reshard_volume (transition.py:153-177) per device; on one GPU it is
reported as bytes and as time at the NVLink 5 per-direction bandwidth.

  python scripts/measure_reshard.py [out.json]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2508_19373_b200.config import get_config, import_moeplan
from paper_2508_19373_b200.layout import PlanDegrees, RankLayout
from paper_2508_19373_b200.transition import reshard_pack, reshard_unpack
from paper_2508_19373_b200.weights import pack_rank_weights, synthetic_weights

NVLINK_BPS = 900e9  # NVLink 5, per direction per GPU (guide figure, not measured here: one-GPU box)


KERNEL_MS = []
TIME_KERNEL = [False]


def _timed_copy_records(recs):
    """ops.copy_records with CUDA events around the one batched launch (second pass only)."""
    if not TIME_KERNEL[0]:
        return ORIG_COPY_RECORDS(recs)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)  # keep the GPU busy while the host submits: s..e is the kernel alone
    s.record()
    out = ORIG_COPY_RECORDS(recs)
    e.record()
    e.synchronize()
    KERNEL_MS.append(s.elapsed_time(e))
    return out


def timed(fn, reps=5):
    """Median wall time of reps calls after one warm call; reps=0: the single first call."""
    if reps == 0:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, out
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2], out


def main():
    global ORIG_COPY_RECORDS
    import paper_2508_19373_b200.ops as ops
    import paper_2508_19373_b200.transition as tr

    ORIG_COPY_RECORDS = ops.copy_records
    ops.copy_records = _timed_copy_records
    mpl = import_moeplan()
    cfg = get_config("mixtral-8x7b")
    spec = cfg.to_model_spec()
    W = synthetic_weights(cfg, "cuda", seed=0)
    N = 8
    rows = []
    for src, dst in (((1, 8), (8, 1)), ((8, 1), (1, 8)), ((2, 4), (8, 1)), ((1, 8), (2, 4))):
        worst = None
        for rank in (0, N - 1):
            mk = lambda te: RankLayout(PlanDegrees(1, N, te[0], te[1], 1), rank, cfg.n_q_heads,  # noqa: E731
                                       cfg.n_kv_heads, cfg.n_experts, cfg.inter, cfg.n_shared)
            li, lj = mk(src), mk(dst)
            wi = pack_rank_weights(cfg, W, li)
            tr._COPY_PLANS.clear()
            tr._STATIC_PLANS.clear()
            t_pack_first, (send, ins, outs, ctx) = timed(lambda: reshard_pack(cfg, wi, li, lj), reps=0)
            recv = torch.randn(sum(outs), device="cuda").to(torch.bfloat16)
            t_unpack_first, _ = timed(lambda: reshard_unpack(ctx, recv), reps=0)
            # every later layer of the switch replays the compiled copy records
            t_pack, (send, ins, outs, ctx) = timed(lambda: reshard_pack(cfg, wi, li, lj))
            t_unpack, _ = timed(lambda: reshard_unpack(ctx, recv))
            TIME_KERNEL[0] = True  # second pass: the batched copy launch alone
            KERNEL_MS.clear()
            timed(lambda: reshard_pack(cfg, wi, li, lj))
            k_pack = sorted(KERNEL_MS)[len(KERNEL_MS) // 2]
            KERNEL_MS.clear()
            timed(lambda: reshard_unpack(ctx, recv))
            k_unpack = sorted(KERNEL_MS)[len(KERNEL_MS) // 2]
            TIME_KERNEL[0] = False
            wj = reshard_unpack(ctx, recv)
            dst_bytes = sum(t.numel() * 2 for t in (wj.w13, wj.w2, wj.ws13, wj.ws2) if t is not None)
            r = {"rank": rank, "pack_ms": t_pack * 1e3, "unpack_ms": t_unpack * 1e3,
                 "first_layer_pack_ms": t_pack_first * 1e3, "first_layer_unpack_ms": t_unpack_first * 1e3,
                 "send_bytes": send.numel() * 2, "recv_bytes": recv.numel() * 2,
                 # HBM bytes each phase moves (read + write): the pieces shipped / the whole destination packing
                 "pack_kernel_ms": k_pack, "unpack_kernel_ms": k_unpack,
                 "pack_kernel_hbm_gbs": 2 * send.numel() * 2 / k_pack / 1e6 if k_pack else 0.0,
                 "unpack_kernel_hbm_gbs": 2 * dst_bytes / k_unpack / 1e6}
            worst = r if worst is None or r["pack_ms"] + r["unpack_ms"] > worst["pack_ms"] + worst["unpack_ms"] else worst
        ref = mpl.reshard_volume(mpl.ExpertStrategy(tp_degree=src[0], ep_degree=src[1]),
                                 mpl.ExpertStrategy(tp_degree=dst[0], ep_degree=dst[1]), spec) / spec.n_layers
        rows.append({"switch": f"exp(tp={src[0]},ep={src[1]}) -> exp(tp={dst[0]},ep={dst[1]})", "n_gpus": N,
                     "reference_reshard_bytes_per_layer": ref, "recv_bytes_rank": worst["recv_bytes"],
                     "pack_ms": worst["pack_ms"], "unpack_ms": worst["unpack_ms"],
                     "first_layer_pack_ms": worst["first_layer_pack_ms"],
                     "first_layer_unpack_ms": worst["first_layer_unpack_ms"],
                     "pack_kernel_ms": worst["pack_kernel_ms"], "unpack_kernel_ms": worst["unpack_kernel_ms"],
                     "pack_kernel_hbm_gbs": worst["pack_kernel_hbm_gbs"],
                     "unpack_kernel_hbm_gbs": worst["unpack_kernel_hbm_gbs"],
                     "transfer_ms_at_nvlink5": worst["recv_bytes"] / NVLINK_BPS * 1e3,
                     "t_reshard_ms_per_layer": worst["pack_ms"] + worst["unpack_ms"]
                     + worst["recv_bytes"] / NVLINK_BPS * 1e3,
                     "reference_t_reshard_ms_per_layer_at_nvlink5": ref / NVLINK_BPS * 1e3})
    out = {"workload": "Mixtral-8x7B, one layer's expert weights (1.41 G params bf16), N=8 layouts, worst of ranks 0/7",
           "note": "pack/unpack measured on one B200 (pack_ms / unpack_ms: wall clock around each phase of a layer that replays the compiled copy records, median of 5; first_layer_*: the first layer of a switch, which plans and compiles them; *_kernel_ms: CUDA events around the phase's one hap_copy2d_batched launch, HBM GB/s = read + write bytes over it); the all-to-all is the reference's volume "
                   "at NVLink 5 900 GB/s (a multi-GPU box is needed to time it)", "rows": rows}
    text = json.dumps(out, indent=1)
    print(text)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(text)


if __name__ == "__main__":
    main()
