"""ctypes binding of ``libhap_kernels.so`` (the C-ABI in include/hap_kernels.h).

The library is REQUIRED: there is no CPU or PyTorch fallback for any op.
Loading fails loudly if the shared object is missing; status codes map to the
reference's exception classes (``SpecError`` is a ValueError subclass in
moeplan/arch.py:12, so argument errors surface as ValueError; device errors as
RuntimeError).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from ._build import LIB_PATH

c_void_p = ctypes.c_void_p
c_int64 = ctypes.c_int64
c_int32 = ctypes.c_int32
c_float = ctypes.c_float
c_size_t = ctypes.c_size_t

HAP_OK = 0
HAP_ERR_INVALID_ARG = -1
HAP_ERR_UNSUPPORTED = -2
HAP_ERR_MISALIGNED = -3
HAP_ERR_LAUNCH = -4
HAP_ERR_WORKSPACE = -5
HAP_ERR_DRIVER = -6

HAP_EPI_STORE = 0
HAP_EPI_SWIGLU = 1
HAP_EPI_F32 = 2

# name -> (restype, argtypes); must mirror include/hap_kernels.h exactly.
SIGNATURES = {
    "hap_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "hap_abi_version": (ctypes.c_int, []),
    "hap_enable_peer_access": (ctypes.c_int, [ctypes.c_int]),
    "hap_swiglu_half_width": (c_int64, [c_int64]),
    "hap_grouped_gemm_bf16": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
         c_void_p, c_int64, c_int32, c_int64, c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "hap_gemm_qkv_rope": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
         c_int64, c_int64, c_float, c_void_p],
    ),
    "hap_gemm_splitk_workspace_bytes": (c_size_t, []),
    "hap_grouped_gemm_bf16_ex": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
         c_void_p, c_int64, c_int32, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_size_t, c_void_p],
    ),
    "hap_grouped_gemm_bf16_sms": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
         c_void_p, c_int64, c_int32, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_size_t, c_int32, c_void_p],
    ),
    "hap_gemm_qkv_rope_ex": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
         c_int64, c_int64, c_float, c_void_p, c_size_t, c_void_p],
    ),
    "hap_grouped_gemm_bf16_scatter": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
         c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "hap_peer_copy_rows": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "hap_peer_allreduce_sig_bytes": (c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "hap_nvls_allreduce_bytes": (c_size_t, [c_int64, ctypes.c_int32]),
    "hap_nvls_allreduce_bf16": (
        ctypes.c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, ctypes.c_int32, ctypes.c_int32, c_void_p],
    ),
    "hap_peer_allreduce_bf16": (
        ctypes.c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, c_void_p],
    ),
    "hap_router_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int32]),
    "hap_router_topk": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64, c_int32, c_int32, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    ),
    "hap_moe_permute_workspace_bytes": (c_size_t, [c_int64, c_int64]),
    "hap_moe_permute": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
         c_size_t, c_void_p],
    ),
    "hap_moe_combine": (
        ctypes.c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p],
    ),
    "hap_moe_combine_chunked": (
        ctypes.c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_int64, c_int64, c_void_p],
    ),
    "hap_rmsnorm": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_float, c_void_p, c_int64, c_void_p],
    ),
    "hap_rmsnorm_multi": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_float, c_void_p, ctypes.c_int32, c_int64, c_void_p],
    ),
    "hap_peer_barrier": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_int32, ctypes.c_int32, c_void_p]),
    "hap_reduce_slots_bf16": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "hap_peer_broadcast_i32": (ctypes.c_int, [c_void_p, c_int64, c_void_p, ctypes.c_int32, c_int64, c_void_p]),
    "hap_ep_exchange_plan": (
        ctypes.c_int,
        [c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "hap_rope_qk": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_float, c_void_p],
    ),
    "hap_attn_prefill_workspace_bytes": (c_size_t, []),
    "hap_attn_prefill": (
        ctypes.c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
         c_int64, c_int64, c_int64, c_float, c_int32, c_void_p, c_size_t, c_void_p],
    ),
    "hap_kv_cache_fill": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "hap_int4_dequant": (
        ctypes.c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int32, c_void_p],
    ),
    "hap_attn_decode_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64]),
    "hap_copy2d_batched": (ctypes.c_int, [c_void_p, c_int64, c_void_p]),
    "hap_rmsnorm_gemm_qkv_rope": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_float, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
         c_void_p, c_int64, c_void_p, c_int64, c_int64, c_float, c_void_p, c_size_t, c_void_p],
    ),
    "hap_kv_cache_fill_paged": (
        ctypes.c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
         c_int64, c_void_p],
    ),
    "hap_attn_decode_paged": (
        ctypes.c_int,
        [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
         c_int64, c_int64, c_float, c_void_p, c_int64, c_void_p, c_size_t, c_void_p],
    ),
    "hap_attn_decode": (
        ctypes.c_int,
        [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64,
         c_float, c_void_p, c_int64, c_void_p, c_size_t, c_void_p],
    ),
}


class HapError(RuntimeError):
    """Device-side failure reported by the kernel library."""


class HapArgumentError(ValueError):
    """Argument rejected by the kernel library before launch."""


_LIB = None


def lib_path() -> Path:
    return Path(os.environ.get("HAP_KERNELS_LIB", str(LIB_PATH)))


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the kernel library; raises if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = Path(path) if path else lib_path()
    if not p.exists():
        raise ImportError(
            f"{p} not found: build the sm_100a kernels first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no fallback path"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(status: int, what: str) -> None:
    if status == HAP_OK:
        return
    msg = load().hap_status_string(status).decode()
    if status in (HAP_ERR_INVALID_ARG, HAP_ERR_UNSUPPORTED, HAP_ERR_MISALIGNED, HAP_ERR_WORKSPACE):
        raise HapArgumentError(f"{what}: {msg} (status {status})")
    raise HapError(f"{what}: {msg} (status {status})")
