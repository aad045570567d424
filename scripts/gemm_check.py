"""Quick GPU check of the tcgen05 grouped GEMM against torch (dev script)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2508_19373_b200._build import LIB_PATH

lib = ctypes.CDLL(str(LIB_PATH))
f = lib.hap_grouped_gemm_bf16
V, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
f.argtypes = [V, I64, I64, I64, V, I64, I64, V, V, I64, I32, I64, V, V, I64, V]
f.restype = ctypes.c_int


def run(A, B, n_groups, N, seg, C, epi=0, hw=0, bias=None, resid=None):
    st = torch.cuda.current_stream().cuda_stream
    r = f(A.data_ptr(), A.shape[0], A.stride(0), A.shape[1], B.data_ptr(), n_groups, N,
          seg.data_ptr() if seg is not None else None, C.data_ptr(), C.stride(0), epi, hw,
          bias.data_ptr() if bias is not None else None, resid.data_ptr() if resid is not None else None,
          resid.stride(0) if resid is not None else 0, st)
    assert r == 0, r


def ref_grouped(A, B, seg, N, epi, hw):
    out = []
    for g in range(len(seg) - 1):
        a = A[seg[g]:seg[g + 1]].float()
        b = B[g * N:(g + 1) * N].float()
        y = a @ b.t()
        if epi == 1:
            nb = N // (2 * hw)
            y = y.view(-1, nb, 2, hw)
            y = torch.nn.functional.silu(y[:, :, 0]) * y[:, :, 1]
            y = y.reshape(-1, N // 2)
        out.append(y)
    return torch.cat(out)


def check(name, got, ref):
    err = (got.float() - ref).abs().max().item()
    rel = err / ref.abs().max().item()
    print(f"{name}: max abs err {err:.4g} rel {rel:.3g}", flush=True)
    return rel


torch.manual_seed(0)
dev = "cuda"
ok = True
# 1) dense single group
for (M, N, K) in [(128, 256, 64), (256, 512, 128), (1000, 768, 4096), (77, 4096, 512)]:
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    run(A, B, 1, N, None, C)
    torch.cuda.synchronize()
    ok &= check(f"dense M={M} N={N} K={K}", C, A.float() @ B.float().t()) < 1e-2

# 2) grouped with ragged segments + swiglu
E, N, K = 8, 512, 1024
counts = torch.tensor([0, 130, 1, 257, 64, 0, 300, 128])
seg = torch.zeros(E + 1, dtype=torch.int32)
seg[1:] = torch.cumsum(counts, 0)
R = int(seg[-1])
A = torch.randn(R, K, device=dev).bfloat16()
B = (torch.randn(E * N, K, device=dev) * 0.05).bfloat16()
segd = seg.to(dev)
C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
run(A, B, E, N, segd, C)
torch.cuda.synchronize()
ok &= check("grouped store", C, ref_grouped(A, B, seg.tolist(), N, 0, 0)) < 1e-2
C2 = torch.zeros(R, N // 2, device=dev, dtype=torch.bfloat16)
run(A, B, E, N, segd, C2, epi=1, hw=128)
torch.cuda.synchronize()
ok &= check("grouped swiglu", C2, ref_grouped(A, B, seg.tolist(), N, 1, 128)) < 2e-2

# 3) bias + residual
M, N, K = 300, 768, 256
A = torch.randn(M, K, device=dev).bfloat16()
B = torch.randn(N, K, device=dev).bfloat16()
bias = torch.randn(N, device=dev).bfloat16()
res = torch.randn(M, N, device=dev).bfloat16()
C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
run(A, B, 1, N, None, C, bias=bias, resid=res)
torch.cuda.synchronize()
ok &= check("bias+resid", C, A.float() @ B.float().t() + bias.float() + res.float()) < 1e-2

# 4) perf: Mixtral gate/up grouped, 8 experts x 4096 rows, N=28672, K=4096
E, M_e, N, K = 8, 4096, 28672, 4096
seg = torch.arange(0, (E + 1) * M_e, M_e, dtype=torch.int32, device=dev)
A = torch.randn(E * M_e, K, device=dev).bfloat16()
B = (torch.randn(E * N, K, device=dev) * 0.02).bfloat16()
C = torch.empty(E * M_e, N // 2, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    run(A, B, E, N, seg, C, epi=1, hw=128)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(10):
    run(A, B, E, N, seg, C, epi=1, hw=128)
t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / 10
fl = 2 * E * M_e * N * K
print(f"gate/up grouped: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
# cuBLAS comparison (dense, same flops)
A2 = A[:M_e]; B2 = B[:N]
t0.record()
for _ in range(10):
    for e in range(E):
        torch.matmul(A2, B2.t())
t1.record(); torch.cuda.synchronize()
ms2 = t0.elapsed_time(t1) / 10
print(f"cuBLAS 8x dense: {ms2:.3f} ms  {fl / ms2 / 1e9:.1f} TFLOP/s", flush=True)
print("ALL OK" if ok else "FAILED")
