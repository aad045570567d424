"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/hap_kernels.h declares with the argument counts the ctypes
table uses, and rejects bad arguments before any launch (no GPU needed)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hap_kernels.h"


def header_functions():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\n(?:const char\*|int64_t|size_t|int)\s+(hap_\w+)\(([^;]*?)\);", src):
        args = [a for a in m.group(2).replace("\n", " ").split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


@pytest.fixture(scope="module")
def lib():
    from paper_2508_19373_b200 import _build, _lib

    _build.build()
    return _lib.load()


def test_every_header_symbol_exported(lib):
    from paper_2508_19373_b200 import _lib

    funcs = header_functions()
    assert len(funcs) >= 13
    nm = subprocess.run(["nm", "-D", str(_lib.lib_path())], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hap_\w+)", nm))
    assert set(funcs) <= exported, set(funcs) - exported
    for name, n_args in funcs.items():
        assert name in _lib.SIGNATURES, name
        assert len(_lib.SIGNATURES[name][1]) == n_args, (name, n_args)


def test_sm100a_code_in_library():
    from paper_2508_19373_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.lib_path())], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "UTCHMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass                         # TMA loads
    assert "LDTM" in sass                            # tcgen05.ld (TMEM -> registers)


def test_status_strings_and_version(lib):
    assert lib.hap_abi_version() == 2
    assert lib.hap_status_string(0) == b"ok"
    assert b"workspace" in lib.hap_status_string(-5)


def test_argument_errors_before_launch(lib):
    # NULL operands / bad shapes are rejected with HAP_ERR_INVALID_ARG (-1) etc.
    assert lib.hap_grouped_gemm_bf16(None, 16, 64, 64, None, 1, 64, None, 1, None, None, 64, 0, 0, None, None, 0,
                                     None) == -1
    # misaligned leading dimension
    p = ctypes.c_void_p(16)
    assert lib.hap_grouped_gemm_bf16(p, 16, 60, 60, p, 1, 64, None, 1, None, p, 64, 0, 0, None, None, 0, None) == -3
    # swiglu half width must divide N/2-blocks
    assert lib.hap_grouped_gemm_bf16(p, 16, 64, 64, p, 1, 96, None, 1, None, p, 64, 1, 64, None, None, 0,
                                     None) == -1
    # router: top_k > n_experts
    assert lib.hap_router_topk(p, 4, 512, p, 2, 3, 1, 0, p, p, None, None, None, 0, None) == -1
    # router: h not a multiple of 64
    assert lib.hap_router_topk(p, 4, 520, p, 8, 2, 1, 0, p, p, None, None, None, 0, None) == -2
    # permute: workspace too small
    assert lib.hap_moe_permute(p, 100, 8, None, 1, 0, None, p, p, p, 4, None) == -5
    # attention: unsupported head_dim
    assert lib.hap_attn_prefill(p, 96 * 3, p, 96 * 3, p, 96 * 3, p, 96, 1, 16, 1, 1, 96, 0.1, 1, p, 8, None) == -2
    # attention: the ticket workspace is the caller's and is required
    assert lib.hap_attn_prefill(p, 384, p, 384, p, 384, p, 128, 1, 16, 1, 1, 128, 0.1, 1, None, 0, None) == -5
    # decode: GQA group larger than 8
    assert lib.hap_attn_decode(p, 4096, p, p, 128, p, 1, 32, 2, 128, 0.1, p, 4096, p, 1 << 20, None) == -2
    # rope gemm: bad head_dim
    assert lib.hap_gemm_qkv_rope(p, 4, 64, 64, p, 96, None, p, 96, p, 1, 96, 1e6, None) == -2


def test_workspace_queries(lib):
    """The library owns no device state: every scratch is a caller workspace sized by a query."""
    assert lib.hap_attn_prefill_workspace_bytes() == 8
    assert lib.hap_router_workspace_bytes(16, 8, 0) == 0          # <= 8 router rows: per-token kernel
    assert lib.hap_router_workspace_bytes(2048, 64, 1) == 0       # large T: TMA router, no scratch
    assert lib.hap_router_workspace_bytes(1, 64, 1) == 4096 + 80 * 4
    assert lib.hap_router_workspace_bytes(1024, 71, 1) == 4096 + 1024 * 80 * 4
    assert lib.hap_gemm_splitk_workspace_bytes() == 32 << 20


def test_swiglu_half_width_rule(lib):
    from paper_2508_19373_b200.weights import swiglu_half_width

    for inter in (14336, 1792, 1408, 704, 352, 176, 2560, 320, 16384, 2048, 5632, 20480):
        assert lib.hap_swiglu_half_width(inter) == swiglu_half_width(inter)
    assert lib.hap_swiglu_half_width(12) == -1


def test_product_path_has_no_cpu_fallback():
    """The executor's compute backend refuses to run without CUDA (no silent fallback)."""
    import torch

    from paper_2508_19373_b200.executor import CudaOps

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU path"):
        CudaOps()
    from paper_2508_19373_b200 import ops

    with pytest.raises(ValueError, match="CUDA tensor"):
        ops.rmsnorm(torch.zeros(2, 64, dtype=torch.bfloat16), torch.ones(64, dtype=torch.bfloat16), 1e-5)
