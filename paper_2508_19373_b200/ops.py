"""Torch-facing wrappers of the C-ABI kernels (include/hap_kernels.h).

Each wrapper validates dtypes / devices / contiguity, passes raw device
pointers plus ``torch.cuda.current_stream()`` to the library and maps status
codes to exceptions.  Nothing here computes on the host and nothing falls
back to PyTorch math: if the library is missing, ``_lib.load`` raises.
"""

from __future__ import annotations

import os
from typing import Optional, Tuple

import torch

from . import _lib
from ._lib import HAP_EPI_F32, HAP_EPI_STORE, HAP_EPI_SWIGLU, check

BF16 = torch.bfloat16

# Kernel launches issued through this module (the bench's gpu_launches claim).
LAUNCHES = [0]


def _count(n: int = 1) -> None:
    LAUNCHES[0] += n


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor, name: str, dtype=None, cuda=True):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def _rowmajor(t: torch.Tensor, name: str):
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D row-major view")


# Caller-owned workspaces of the C-ABI (the library keeps no device state):
# one per (kind, device, stream), allocated once at its maximum size and never
# reallocated, so CUDA graphs that captured a launch keep a valid pointer and
# launches on different streams never share scratch.  The self-resetting
# workspaces (attention tickets, router counters) are zero-filled once here.
# SPLITK[0] = False runs the plain GEMM entry points (A/B experiments, tests).
SPLITK = [os.environ.get("HAP_GEMM_SPLITK", "1") != "0"]
_WS = {}
_ROUTER_MAX_T, _ROUTER_MAX_ROWS = 1024, 72


def stream_workspace(kind: str, device: torch.device) -> torch.Tensor:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (kind, idx, _stream())
    ws = _WS.get(key)
    if ws is None:
        lib = _lib.load()
        if kind == "splitk":
            n, zero = int(lib.hap_gemm_splitk_workspace_bytes()), False
        elif kind == "attn":
            n, zero = int(lib.hap_attn_prefill_workspace_bytes()), True
        elif kind == "router":
            n, zero = int(lib.hap_router_workspace_bytes(_ROUTER_MAX_T, _ROUTER_MAX_ROWS - 1, 1)), True
        else:
            raise ValueError(kind)
        dev = torch.device("cuda", idx)
        ws = torch.zeros(n, device=dev, dtype=torch.uint8) if zero else torch.empty(n, device=dev, dtype=torch.uint8)
        _WS[key] = ws
    return ws


def splitk_workspace(device: torch.device) -> Tuple[int, int]:
    if not SPLITK[0]:
        return 0, 0
    ws = stream_workspace("splitk", device)
    return ws.data_ptr(), ws.numel()


def swiglu_half_width(inter: int) -> int:
    hw = _lib.load().hap_swiglu_half_width(int(inter))
    if hw <= 0:
        raise ValueError(f"no SwiGLU tile width divides inter={inter}")
    return int(hw)


def grouped_gemm(a: torch.Tensor, b: torch.Tensor, n_groups: int, seg: Optional[torch.Tensor],
                 out: torch.Tensor, *, swiglu_half: int = 0, bias: Optional[torch.Tensor] = None,
                 residual: Optional[torch.Tensor] = None,
                 seg_group: Optional[torch.Tensor] = None, sm_budget: int = 0) -> torch.Tensor:
    """out[r] = epi(a[r] @ b[g*N:(g+1)*N]^T) for rows r of segment s, g = seg_group[s] (tcgen05 kernel).

    A float32 ``out`` selects HAP_EPI_F32: the unrounded fp32 accumulators
    (no bias / residual / SwiGLU), the fp32-accumulate parity check.
    ``sm_budget`` > 0 keeps the launch on at most that many SMs
    (hap_grouped_gemm_bf16_sms), for weight streams running beside others."""
    lib = _lib.load()
    f32 = out.dtype == torch.float32
    _need(a, "a", BF16); _need(b, "b", BF16); _need(out, "out", torch.float32 if f32 else BF16)
    _rowmajor(a, "a"); _rowmajor(out, "out")
    if not b.is_contiguous():
        raise ValueError("b must be contiguous [n_groups*N, K]")
    K = a.shape[1]
    b2 = b.reshape(-1, b.shape[-1])
    if b2.shape[1] != K or b2.shape[0] % n_groups:
        raise ValueError(f"b shape {tuple(b.shape)} incompatible with K={K}, n_groups={n_groups}")
    N = b2.shape[0] // n_groups
    n_segs = 1
    if seg is not None:
        _need(seg, "seg", torch.int32)
        n_segs = seg.numel() - 1
        if seg_group is not None:
            _need(seg_group, "seg_group", torch.int32)
            if seg_group.numel() != n_segs:
                raise ValueError("seg_group must have one entry per segment")
        elif n_segs != n_groups:
            raise ValueError("seg must have n_groups+1 entries (or pass seg_group)")
    elif n_groups != 1:
        raise ValueError("seg is required when n_groups > 1")
    epi = HAP_EPI_SWIGLU if swiglu_half else HAP_EPI_STORE
    if f32:
        if swiglu_half or bias is not None or residual is not None:
            raise ValueError("a float32 out takes the raw accumulators: no SwiGLU, bias or residual")
        epi = HAP_EPI_F32
    if residual is not None:
        _need(residual, "residual", BF16); _rowmajor(residual, "residual")
    if bias is not None:
        _need(bias, "bias", BF16)
    ws, ws_bytes = splitk_workspace(a.device)
    st = lib.hap_grouped_gemm_bf16_sms(a.data_ptr(), a.shape[0], a.stride(0), K, b2.data_ptr(), n_groups, N,
                                       _ptr(seg), n_segs, _ptr(seg_group), out.data_ptr(), out.stride(0), epi,
                                       int(swiglu_half),
                                       _ptr(bias), _ptr(residual), residual.stride(0) if residual is not None else 0,
                                       ws or None, ws_bytes, int(sm_budget), _stream())
    check(st, "hap_grouped_gemm_bf16_sms")
    _count(1 if a.shape[0] else 0)
    return out


def grouped_gemm_scatter(a: torch.Tensor, b: torch.Tensor, n_groups: int, seg: torch.Tensor,
                         seg_group: Optional[torch.Tensor], seg_dst: torch.Tensor, seg_dst_row0: torch.Tensor,
                         ldc: int) -> None:
    """Grouped GEMM (store epilogue) whose rows of segment s land at
    seg_dst[s] + (r - seg[s] + seg_dst_row0[s]) * ldc (device addresses, e.g.
    peer-mapped buffers): the EP combine fused into the down projection."""
    lib = _lib.load()
    _need(a, "a", BF16); _need(b, "b", BF16); _rowmajor(a, "a")
    _need(seg, "seg", torch.int32); _need(seg_dst, "seg_dst", torch.int64); _need(seg_dst_row0, "seg_dst_row0", torch.int32)
    K = a.shape[1]
    b2 = b.reshape(-1, b.shape[-1])
    N = b2.shape[0] // n_groups
    n_segs = seg.numel() - 1
    if seg_dst.numel() != n_segs or seg_dst_row0.numel() != n_segs:
        raise ValueError("seg_dst / seg_dst_row0 need one entry per segment")
    if seg_group is not None:
        _need(seg_group, "seg_group", torch.int32)
    st = lib.hap_grouped_gemm_bf16_scatter(a.data_ptr(), a.shape[0], a.stride(0), K, b2.data_ptr(), n_groups, N,
                                           seg.data_ptr(), n_segs, _ptr(seg_group), seg_dst.data_ptr(),
                                           seg_dst_row0.data_ptr(), ldc, _stream())
    check(st, "hap_grouped_gemm_bf16_scatter")
    _count(1 if a.shape[0] else 0)


def peer_copy_rows(src: torch.Tensor, seg: torch.Tensor, dst_base: torch.Tensor, dst_row0: torch.Tensor,
                   ldd: int) -> None:
    """Copy the row segments of src to (peer) addresses dst_base[s] + (dst_row0[s] + i) * ldd."""
    lib = _lib.load()
    _need(src, "src", BF16); _rowmajor(src, "src")
    if src.stride(0) != src.shape[1]:
        raise ValueError("src must be contiguous")
    _need(seg, "seg", torch.int32); _need(dst_base, "dst_base", torch.int64); _need(dst_row0, "dst_row0", torch.int64)
    st = lib.hap_peer_copy_rows(src.data_ptr(), src.shape[0], src.shape[1], seg.data_ptr(), seg.numel() - 1,
                                dst_base.data_ptr(), dst_row0.data_ptr(), ldd, _stream())
    check(st, "hap_peer_copy_rows")
    _count(1 if src.shape[0] else 0)


def peer_allreduce(in_ptrs: torch.Tensor, out_ptrs: torch.Tensor, epoch_ptrs: torch.Tensor, data_ptrs: torch.Tensor,
                   sig_ptrs: torch.Tensor, n: int, n_max: int, n_ranks: int, rank0: int, ranks_in_launch: int,
                   n_ctas: int) -> None:
    """One-shot all-reduce over peer-mapped memory (tables of device addresses, see hap_kernels.h)."""
    lib = _lib.load()
    for t, name in ((in_ptrs, "in_ptrs"), (out_ptrs, "out_ptrs"), (epoch_ptrs, "epoch_ptrs"),
                    (data_ptrs, "data_ptrs"), (sig_ptrs, "sig_ptrs")):
        _need(t, name, torch.int64)
    st = lib.hap_peer_allreduce_bf16(in_ptrs.data_ptr(), out_ptrs.data_ptr(), epoch_ptrs.data_ptr(),
                                     data_ptrs.data_ptr(), sig_ptrs.data_ptr(), n, n_max, n_ranks, rank0,
                                     ranks_in_launch, n_ctas, _stream())
    check(st, "hap_peer_allreduce_bf16")
    _count(1 if n else 0)


def gemm(a: torch.Tensor, w: torch.Tensor, out: Optional[torch.Tensor] = None, *, bias=None, residual=None,
         swiglu_half: int = 0, sm_budget: int = 0) -> torch.Tensor:
    """Dense a @ w^T (nn.Linear layout) on the tcgen05 kernel."""
    n_out = w.shape[0] // 2 if swiglu_half else w.shape[0]
    if out is None:
        out = torch.empty(a.shape[0], n_out, device=a.device, dtype=BF16)
    return grouped_gemm(a, w, 1, None, out, swiglu_half=swiglu_half, bias=bias, residual=residual,
                        sm_budget=sm_budget)


def gemm_qkv_rope(a: torch.Tensor, w: torch.Tensor, positions: torch.Tensor, n_rope_heads: int, head_dim: int,
                  theta: float, bias: Optional[torch.Tensor] = None,
                  out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """qkv = a @ w^T (+bias) with RoPE applied to the first n_rope_heads heads (fused epilogue)."""
    lib = _lib.load()
    _need(a, "a", BF16); _need(w, "w", BF16); _need(positions, "positions", torch.int32)
    _rowmajor(a, "a")
    if not w.is_contiguous():
        raise ValueError("w must be contiguous")
    if bias is not None:
        _need(bias, "bias", BF16)
    N = w.shape[0]
    if out is None:
        out = torch.empty(a.shape[0], N, device=a.device, dtype=BF16)
    _need(out, "out", BF16); _rowmajor(out, "out")
    ws, ws_bytes = splitk_workspace(a.device)
    st = lib.hap_gemm_qkv_rope_ex(a.data_ptr(), a.shape[0], a.stride(0), a.shape[1], w.data_ptr(), N, _ptr(bias),
                                  out.data_ptr(), out.stride(0), positions.data_ptr(), n_rope_heads, head_dim,
                                  float(theta), ws or None, ws_bytes, _stream())
    check(st, "hap_gemm_qkv_rope_ex")
    _count(1 if a.shape[0] else 0)
    return out


_HN_SCRATCH: dict = {}


def rmsnorm_qkv_rope(x: torch.Tensor, norm_w: torch.Tensor, eps: float, w: torch.Tensor, positions: torch.Tensor,
                     n_rope_heads: int, head_dim: int, theta: float, bias: Optional[torch.Tensor] = None,
                     out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm_qkv_rope(rmsnorm(x, norm_w, eps), ...) through hap_rmsnorm_gemm_qkv_rope:
    one launch at decode sizes (the GEMV normalises while staging its rows),
    bit-identical to the two calls."""
    lib = _lib.load()
    _need(x, "x", BF16); _need(norm_w, "norm_w", BF16); _need(w, "w", BF16)
    _need(positions, "positions", torch.int32)
    _rowmajor(x, "x")
    if not w.is_contiguous() or not norm_w.is_contiguous():
        raise ValueError("w and norm_w must be contiguous")
    if bias is not None:
        _need(bias, "bias", BF16)
    M, K = x.shape
    N = w.shape[0]
    if out is None:
        out = torch.empty(M, N, device=x.device, dtype=BF16)
    _need(out, "out", BF16); _rowmajor(out, "out")
    if M <= 2:  # the GEMV path never writes hn: a persistent scratch per stream, no allocation per call
        key = (x.device, K, _stream())
        hn = _HN_SCRATCH.get(key)
        if hn is None:
            hn = _HN_SCRATCH[key] = torch.empty(2, K, device=x.device, dtype=BF16)
        hn = hn[:M]
    else:
        hn = torch.empty(M, K, device=x.device, dtype=BF16)
    ws, ws_bytes = splitk_workspace(x.device)
    st = lib.hap_rmsnorm_gemm_qkv_rope(x.data_ptr(), M, x.stride(0), K, norm_w.data_ptr(), float(eps),
                                       hn.data_ptr(), hn.stride(0), w.data_ptr(), N, _ptr(bias), out.data_ptr(),
                                       out.stride(0), positions.data_ptr(), n_rope_heads, head_dim, float(theta),
                                       ws or None, ws_bytes, _stream())
    check(st, "hap_rmsnorm_gemm_qkv_rope")
    _count(1 if M <= 2 else 2)
    return out


def router_topk(x: torch.Tensor, w: torch.Tensor, n_experts: int, top_k: int, renormalize: bool,
                has_shared_gate: bool, topk_idx: torch.Tensor, topk_w: torch.Tensor,
                shared_gate: Optional[torch.Tensor] = None, logits: Optional[torch.Tensor] = None,
                workspace: Optional[torch.Tensor] = None):
    """Fixed-order fp32 router logits -> top-k (hap_router_topk).  workspace:
    zero-filled uint8 scratch (default: this stream's cached one)."""
    lib = _lib.load()
    ws = workspace if workspace is not None else stream_workspace("router", x.device)
    _need(x, "x", BF16); _need(w, "w", BF16)
    if not x.is_contiguous() or not w.is_contiguous():
        raise ValueError("router inputs must be contiguous")
    _need(topk_idx, "topk_idx", torch.int32); _need(topk_w, "topk_w", torch.float32)
    st = lib.hap_router_topk(x.data_ptr(), x.shape[0], x.shape[1], w.data_ptr(), n_experts, top_k,
                             int(renormalize), int(has_shared_gate), topk_idx.data_ptr(), topk_w.data_ptr(),
                             _ptr(shared_gate), _ptr(logits), ws.data_ptr(), ws.numel(), _stream())
    check(st, "hap_router_topk")
    _count(1 if x.shape[0] else 0)


def permute_workspace_bytes(rows: int, n_experts: int) -> int:
    return int(_lib.load().hap_moe_permute_workspace_bytes(rows, n_experts))


def moe_permute(expert_of_row: torch.Tensor, n_experts: int, x: Optional[torch.Tensor], src_row_div: int,
                x_out: Optional[torch.Tensor], dst_of_row: torch.Tensor, seg: torch.Tensor,
                workspace: torch.Tensor) -> None:
    lib = _lib.load()
    _need(expert_of_row, "expert_of_row", torch.int32)
    _need(dst_of_row, "dst_of_row", torch.int32); _need(seg, "seg", torch.int32)
    R = expert_of_row.numel()
    h = 0
    if x_out is not None:
        _need(x, "x", BF16); _need(x_out, "x_out", BF16)
        if not x.is_contiguous() or not x_out.is_contiguous():
            raise ValueError("permute payloads must be contiguous")
        h = x.shape[1]
    st = lib.hap_moe_permute(expert_of_row.data_ptr(), R, n_experts, _ptr(x), src_row_div, h, _ptr(x_out),
                             dst_of_row.data_ptr(), seg.data_ptr(), workspace.data_ptr(),
                             workspace.numel() * workspace.element_size(), _stream())
    check(st, "hap_moe_permute")
    _count((3 if R > 512 else 2) if R else 0)  # rank (+ scan when > 1 block of 512 rows) + scatter


def moe_combine(y: torch.Tensor, dst_of_row: torch.Tensor, topk_w: torch.Tensor, T: int, k: int,
                out: torch.Tensor, residual: Optional[torch.Tensor] = None,
                shared_y: Optional[torch.Tensor] = None, shared_gate: Optional[torch.Tensor] = None,
                res_row0: int = 0, res_rows: Optional[int] = None) -> None:
    """out[t] = sum_j w * y[dst] (+ sg * shared_y) (+ residual[t - res_row0] inside the row window)."""
    lib = _lib.load()
    _need(y, "y", BF16); _need(out, "out", BF16)
    for t, n in ((y, "y"), (out, "out"), (residual, "residual"), (shared_y, "shared_y")):
        if t is not None and not t.is_contiguous():
            raise ValueError(f"{n} must be contiguous")
    h = out.shape[1]
    if residual is not None and res_rows is None:
        res_rows = residual.shape[0]
    st = lib.hap_moe_combine(y.data_ptr(), dst_of_row.data_ptr(), topk_w.data_ptr(), T, k, h, _ptr(residual),
                             int(res_row0), int(res_rows or 0), _ptr(shared_y), _ptr(shared_gate), out.data_ptr(),
                             _stream())
    check(st, "hap_moe_combine")
    _count(1 if T else 0)


def moe_combine_chunked(y: torch.Tensor, dst_of_row: torch.Tensor, topk_w: torch.Tensor, T: int, k: int, h: int,
                        dst_tab: torch.Tensor, chunk_rows: int, slot: int, residual: Optional[torch.Tensor] = None,
                        shared_y: Optional[torch.Tensor] = None, shared_gate: Optional[torch.Tensor] = None,
                        res_row0: int = 0, res_rows: Optional[int] = None) -> None:
    """moe_combine whose chunk q of rows is stored into slot `slot` of the buffer
    dst_tab[q] (device int64 table of peer-mapped bases): the pushed reduce-scatter."""
    lib = _lib.load()
    _need(y, "y", BF16); _need(dst_tab, "dst_tab", torch.int64)
    for t, n in ((y, "y"), (residual, "residual"), (shared_y, "shared_y")):
        if t is not None and not t.is_contiguous():
            raise ValueError(f"{n} must be contiguous")
    if residual is not None and res_rows is None:
        res_rows = residual.shape[0]
    st = lib.hap_moe_combine_chunked(y.data_ptr(), dst_of_row.data_ptr(), topk_w.data_ptr(), T, k, h,
                                     _ptr(residual), int(res_row0), int(res_rows or 0), _ptr(shared_y),
                                     _ptr(shared_gate), dst_tab.data_ptr(), int(chunk_rows), int(slot), _stream())
    check(st, "hap_moe_combine_chunked")
    _count(1 if T else 0)


def rmsnorm_multi(x: torch.Tensor, w: torch.Tensor, eps: float, dst_tab: torch.Tensor, ldo: int) -> None:
    """RMSNorm storing every row to each base of dst_tab (the pushed all-gather)."""
    lib = _lib.load()
    _need(x, "x", BF16); _need(w, "w", BF16); _need(dst_tab, "dst_tab", torch.int64)
    _rowmajor(x, "x")
    st = lib.hap_rmsnorm_multi(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), w.data_ptr(), float(eps),
                               dst_tab.data_ptr(), dst_tab.numel(), int(ldo), _stream())
    check(st, "hap_rmsnorm_multi")
    _count(1 if x.shape[0] else 0)


def peer_barrier(sig_tab: torch.Tensor, epoch: torch.Tensor, n_ranks: int, rank: int) -> None:
    """Device-side barrier of a peer group (no host synchronisation)."""
    lib = _lib.load()
    _need(sig_tab, "sig_tab", torch.int64); _need(epoch, "epoch", torch.int32)
    check(lib.hap_peer_barrier(sig_tab.data_ptr(), epoch.data_ptr(), n_ranks, rank, _stream()), "hap_peer_barrier")
    _count(1)


def reduce_slots(slots: torch.Tensor, n_slots: int, rows: int, out: torch.Tensor) -> torch.Tensor:
    """out = sum over n_slots row blocks of slots (slot order, fp32, one bf16 rounding)."""
    lib = _lib.load()
    _need(slots, "slots", BF16); _need(out, "out", BF16)
    if not (slots.is_contiguous() and out.is_contiguous()):
        raise ValueError("slots and out must be contiguous")
    h = out.shape[1]
    check(lib.hap_reduce_slots_bf16(slots.data_ptr(), n_slots, rows, h, out.data_ptr(), _stream()),
          "hap_reduce_slots_bf16")
    _count(1 if rows else 0)
    return out


def peer_broadcast_i32(src: torch.Tensor, dst_tab: torch.Tensor, dst_offset_bytes: int) -> None:
    """Push src (int32) to dst_tab[p] + dst_offset_bytes for every base p."""
    lib = _lib.load()
    _need(src, "src", torch.int32); _need(dst_tab, "dst_tab", torch.int64)
    check(lib.hap_peer_broadcast_i32(src.data_ptr(), src.numel(), dst_tab.data_ptr(), dst_tab.numel(),
                                     int(dst_offset_bytes), _stream()), "hap_peer_broadcast_i32")
    _count(1 if src.numel() else 0)


def ep_exchange_plan(segs: torch.Tensor, ep: int, experts_local: int, me: int, dst_row0: torch.Tensor,
                     seg_r: torch.Tensor, seg_dst_row0: torch.Tensor) -> None:
    """Device-side EP dispatch / combine offsets from the gathered segment offsets."""
    lib = _lib.load()
    _need(segs, "segs", torch.int32); _need(dst_row0, "dst_row0", torch.int64)
    _need(seg_r, "seg_r", torch.int32); _need(seg_dst_row0, "seg_dst_row0", torch.int32)
    check(lib.hap_ep_exchange_plan(segs.data_ptr(), ep, experts_local, me, dst_row0.data_ptr(), seg_r.data_ptr(),
                                   seg_dst_row0.data_ptr(), _stream()), "hap_ep_exchange_plan")
    _count(1)


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    lib = _lib.load()
    _need(x, "x", BF16); _need(w, "w", BF16)
    _rowmajor(x, "x")
    if out is None:
        out = torch.empty(x.shape, device=x.device, dtype=BF16)
    st = lib.hap_rmsnorm(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), w.data_ptr(), float(eps),
                         out.data_ptr(), out.stride(0), _stream())
    check(st, "hap_rmsnorm")
    _count(1 if x.shape[0] else 0)
    return out


def rope_qk(qkv: torch.Tensor, n_q: int, n_kv: int, head_dim: int, positions: torch.Tensor, theta: float):
    lib = _lib.load()
    _need(qkv, "qkv", BF16); _need(positions, "positions", torch.int32)
    _rowmajor(qkv, "qkv")
    st = lib.hap_rope_qk(qkv.data_ptr(), qkv.shape[0], qkv.stride(0), n_q, n_kv, head_dim, positions.data_ptr(),
                         float(theta), _stream())
    check(st, "hap_rope_qk")
    _count(1 if qkv.shape[0] else 0)


def attn_prefill(qkv: torch.Tensor, n_q: int, n_kv: int, head_dim: int, n_seqs: int, seq_len: int,
                 out: torch.Tensor, causal: bool = True, workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Attention over a fused [T, (n_q + 2 n_kv) * d] qkv buffer -> out [T, n_q * d].
    workspace: zero-filled uint8 ticket scratch (default: this stream's cached one)."""
    lib = _lib.load()
    ws = workspace if workspace is not None else stream_workspace("attn", qkv.device)
    _need(qkv, "qkv", BF16); _need(out, "out", BF16)
    _rowmajor(qkv, "qkv"); _rowmajor(out, "out")
    ld = qkv.stride(0)
    base = qkv.data_ptr()
    esz = qkv.element_size()
    st = lib.hap_attn_prefill(base, ld, base + n_q * head_dim * esz, ld, base + (n_q + n_kv) * head_dim * esz, ld,
                              out.data_ptr(), out.stride(0), n_seqs, seq_len, n_q, n_kv, head_dim,
                              float(head_dim ** -0.5), int(causal), ws.data_ptr(), ws.numel(), _stream())
    check(st, "hap_attn_prefill")
    _count(1 if n_seqs * seq_len else 0)
    return out


def kv_cache_fill(qkv: torch.Tensor, n_q: int, n_kv: int, head_dim: int, n_seqs: int, seq_len: int,
                  k_cache: torch.Tensor, v_cache: torch.Tensor) -> None:
    """Write the prefill tokens' k/v (post-RoPE, fused qkv rows) into cache positions [0, seq_len)."""
    lib = _lib.load()
    _need(qkv, "qkv", BF16); _need(k_cache, "k_cache", BF16); _need(v_cache, "v_cache", BF16)
    _rowmajor(qkv, "qkv")
    if k_cache.dim() != 4 or not k_cache.is_contiguous() or not v_cache.is_contiguous():
        raise ValueError("caches must be contiguous [B, n_kv, max_len, d]")
    st = lib.hap_kv_cache_fill(qkv.data_ptr(), qkv.stride(0), n_seqs, seq_len, n_q, n_kv, head_dim,
                               k_cache.data_ptr(), v_cache.data_ptr(), k_cache.shape[2], _stream())
    check(st, "hap_kv_cache_fill")
    _count(1 if n_seqs * seq_len else 0)


def int4_dequant(codes: torch.Tensor, scales: torch.Tensor, zero_points: torch.Tensor, group_size: int, n: int,
                 out: torch.Tensor) -> torch.Tensor:
    """GQI4 dequantization on the GPU: out (float64 -> bit-exact vs moeplan quant.dequantize, or bf16)."""
    lib = _lib.load()
    _need(codes, "codes", torch.uint8); _need(scales, "scales", torch.float64)
    _need(zero_points, "zero_points", torch.float64); _need(out, "out")
    if out.dtype not in (torch.float64, BF16) or out.numel() < n:
        raise ValueError("out must be float64 or bf16 with >= n elements")
    st = lib.hap_int4_dequant(codes.data_ptr(), scales.data_ptr(), zero_points.data_ptr(), int(group_size), int(n),
                              out.data_ptr(), int(out.dtype == BF16), _stream())
    check(st, "hap_int4_dequant")
    _count(1 if n else 0)
    return out


def attn_decode_workspace_bytes(B: int, n_q: int, head_dim: int, max_len: int) -> int:
    return int(_lib.load().hap_attn_decode_workspace_bytes(B, n_q, head_dim, max_len))


def attn_decode(qkv: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, pos: torch.Tensor,
                n_q: int, n_kv: int, head_dim: int, out: torch.Tensor, workspace: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    _need(qkv, "qkv", BF16); _need(k_cache, "k_cache", BF16); _need(v_cache, "v_cache", BF16)
    _need(pos, "pos", torch.int32); _need(out, "out", BF16)
    if k_cache.dim() != 4 or not k_cache.is_contiguous() or not v_cache.is_contiguous():
        raise ValueError("caches must be contiguous [B, n_kv, max_len, d]")
    B, _, max_len, _ = k_cache.shape
    st = lib.hap_attn_decode(qkv.data_ptr(), qkv.stride(0), k_cache.data_ptr(), v_cache.data_ptr(), max_len,
                             pos.data_ptr(), B, n_q, n_kv, head_dim, float(head_dim ** -0.5), out.data_ptr(),
                             out.stride(0), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                             _stream())
    check(st, "hap_attn_decode")
    _count(3 if B else 0)
    return out


def kv_cache_fill_paged(qkv: torch.Tensor, n_q: int, n_kv: int, head_dim: int, n_seqs: int, seq_len: int,
                        k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor) -> None:
    """Prefill k/v into a paged cache: pools [n_pages, n_kv, page, d], int32 block_table [B, max_pages]."""
    lib = _lib.load()
    _need(qkv, "qkv", BF16); _need(k_pool, "k_pool", BF16); _need(v_pool, "v_pool", BF16)
    _need(block_table, "block_table", torch.int32)
    _rowmajor(qkv, "qkv")
    if k_pool.dim() != 4 or not (k_pool.is_contiguous() and v_pool.is_contiguous() and block_table.is_contiguous()):
        raise ValueError("pools must be contiguous [n_pages, n_kv, page, d], block_table contiguous [B, max_pages]")
    st = lib.hap_kv_cache_fill_paged(qkv.data_ptr(), qkv.stride(0), n_seqs, seq_len, n_q, n_kv, head_dim,
                                     k_pool.data_ptr(), v_pool.data_ptr(), block_table.data_ptr(),
                                     block_table.shape[1], k_pool.shape[2], _stream())
    check(st, "hap_kv_cache_fill_paged")
    _count(1 if n_seqs * seq_len else 0)


def attn_decode_paged(qkv: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor, block_table: torch.Tensor,
                      pos: torch.Tensor, n_q: int, n_kv: int, head_dim: int, out: torch.Tensor,
                      workspace: torch.Tensor) -> torch.Tensor:
    """Append + split-KV decode over a paged cache (see hap_attn_decode_paged)."""
    lib = _lib.load()
    _need(qkv, "qkv", BF16); _need(k_pool, "k_pool", BF16); _need(v_pool, "v_pool", BF16)
    _need(block_table, "block_table", torch.int32); _need(pos, "pos", torch.int32); _need(out, "out", BF16)
    if k_pool.dim() != 4 or not (k_pool.is_contiguous() and v_pool.is_contiguous() and block_table.is_contiguous()):
        raise ValueError("pools must be contiguous [n_pages, n_kv, page, d], block_table contiguous [B, max_pages]")
    B = pos.numel()
    st = lib.hap_attn_decode_paged(qkv.data_ptr(), qkv.stride(0), k_pool.data_ptr(), v_pool.data_ptr(),
                                   k_pool.shape[0], k_pool.shape[2], block_table.data_ptr(), block_table.shape[1],
                                   pos.data_ptr(), B, n_q, n_kv, head_dim, float(head_dim ** -0.5), out.data_ptr(),
                                   out.stride(0), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                   _stream())
    check(st, "hap_attn_decode_paged")
    _count(3 if B else 0)
    return out


def nvls_allreduce(inp: torch.Tensor, out: torch.Tensor, uc_base: int, mc_base: int, epoch: torch.Tensor,
                   n_max: int, n_ranks: int, n_ctas: int) -> torch.Tensor:
    """In-switch (NVLS multimem) all-reduce of a bf16 tensor; see hap_nvls_allreduce_bf16."""
    lib = _lib.load()
    _need(inp, "inp", BF16); _need(out, "out", BF16); _need(epoch, "epoch", torch.int32)
    if not (inp.is_contiguous() and out.is_contiguous()):
        raise ValueError("inp and out must be contiguous")
    check(lib.hap_nvls_allreduce_bf16(inp.data_ptr(), out.data_ptr(), uc_base, mc_base, epoch.data_ptr(),
                                      inp.numel(), n_max, n_ranks, n_ctas, _stream()), "hap_nvls_allreduce_bf16")
    _count(1 if inp.numel() else 0)
    return out


def _rows_split(shape, strides_a, strides_b):
    """(rows, row_elems, pitch_a, pitch_b) when both strided views of `shape`
    are `rows` runs of `row_elems` contiguous elements at one uniform pitch
    each (None otherwise).  Trailing dims merge into the row while both views
    stay contiguous; the leading dims must collapse to a single stride."""
    dims = [(s, a, b) for s, a, b in zip(shape, strides_a, strides_b) if s != 1]
    if not dims:
        return 1, 1, 1, 1
    k, inner = len(dims), 1
    while k > 0 and dims[k - 1][1] == inner and dims[k - 1][2] == inner:
        inner *= dims[k - 1][0]
        k -= 1
    if k == 0:
        return 1, inner, inner, inner
    for i in range(k - 1):
        s_next, a_next, b_next = dims[i + 1]
        if dims[i][1] != a_next * s_next or dims[i][2] != b_next * s_next:
            return None
    rows = 1
    for s, _, _ in dims[:k]:
        rows *= s
    return rows, inner, dims[k - 1][1], dims[k - 1][2]


def view_records(pairs):
    """hap_copy2d_batched records (int64 [n, 6]: src, dst, rows, row_bytes,
    src_pitch, dst_pitch) for dst.copy_(src) over same-shape, same-dtype CUDA
    views; each pair must be a uniform-pitch stack of contiguous rows
    (ValueError otherwise — there is no per-pair fallback)."""
    import numpy as np

    recs = []
    for src, dst in pairs:
        _need(src, "src"); _need(dst, "dst", src.dtype)
        if src.shape != dst.shape:
            raise ValueError(f"shape mismatch {tuple(src.shape)} vs {tuple(dst.shape)}")
        if src.numel() == 0:
            continue
        sp = _rows_split(src.shape, src.stride(), dst.stride())
        if sp is None:
            raise ValueError(f"views {tuple(src.stride())} / {tuple(dst.stride())} are not uniform-pitch row stacks")
        rows, inner, ps, pd = sp
        es = src.element_size()
        recs.append((src.data_ptr(), dst.data_ptr(), rows, inner * es, ps * es, pd * es))
    return np.array(recs, dtype=np.int64).reshape(-1, 6)


def copy_records(recs) -> int:
    """One hap_copy2d_batched call over int64 [n, 6] records on the current
    stream; returns the bytes moved."""
    import numpy as np

    lib = _lib.load()
    recs = np.ascontiguousarray(recs, dtype=np.int64)
    if len(recs) == 0:
        return 0
    st = lib.hap_copy2d_batched(recs.ctypes.data, len(recs), _stream())
    check(st, "hap_copy2d_batched")
    _count(-(-len(recs) // 192))
    return int((recs[:, 2] * recs[:, 3]).sum())


def copy_views(pairs) -> int:
    """dst.copy_(src) for every (src, dst) pair in ONE hap_copy2d_batched
    launch (see view_records).  Returns the bytes moved."""
    return copy_records(view_records(pairs))
