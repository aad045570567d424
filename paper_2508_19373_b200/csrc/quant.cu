// INT4 per-group dequantization of the reference's GQI4 container
// (moeplan quant.py:19-22, 61-116): codes packed two per byte, low nibble =
// even index; per group of `group_size` elements a float64 scale and zero
// point; value = code * scale + zero_point.
//
// The fp64 output reproduces quant.py:dequantize bit for bit: the product and
// the sum are rounded separately (__dmul_rn / __dadd_rn, no FMA contraction),
// exactly like numpy's `codes * scales + zero_points`.  The bf16 output is the
// same value rounded to fp32 then to bf16 (the weights the GEMMs consume).
//
// Memory-bound: each thread expands 4 packed bytes (8 elements); the per-group
// scale/zero are read once per group through L1.  Used by the prefill->decode
// weight switch of Eq.6 (transition.py:180-199) to restore
// weights from the INT4 host backup.
#include "common.cuh"

namespace hap {
namespace quant {

constexpr int kThreads = 256;

template <bool kBf16>
__global__ void __launch_bounds__(kThreads) dequant_kernel(const uint8_t* __restrict__ codes,
                                                           const double* __restrict__ scales,
                                                           const double* __restrict__ zeros, int64_t group_size,
                                                           int64_t n, void* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t n8 = (n + 7) / 8;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < n8; v += (int64_t)gridDim.x * kThreads) {
    const int64_t e0 = v * 8;
    const int64_t b0 = v * 4;
    const int64_t nbytes = (n + 1) / 2;
    uint32_t packed = 0;
    if (b0 + 3 < nbytes) {
      packed = *reinterpret_cast<const uint32_t*>(codes + b0);  // 4-byte aligned: b0 % 4 == 0
    } else {
      for (int i = 0; i < 4 && b0 + i < nbytes; ++i) packed |= (uint32_t)codes[b0 + i] << (8 * i);
    }
    double val[8];
    // group of the first / last element (two divisions per 8 elements); the
    // common case (group_size % 8 == 0) has all 8 in one group
    const int64_t g_first = e0 / group_size;
    const int64_t last = (e0 + 7 < n ? e0 + 7 : n - 1);
    const int64_t g_last = last / group_size;
    if (g_first == g_last) {
      const double sc = __ldg(scales + g_first), zp = __ldg(zeros + g_first);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        val[i] = __dadd_rn(__dmul_rn((double)((packed >> (4 * i)) & 0xF), sc), zp);
    } else {
      int64_t g = g_first;
      int64_t next = (g_first + 1) * group_size;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (e0 + i >= next && e0 + i <= last) {
          g = (e0 + i) / group_size;
          next = (g + 1) * group_size;
        }
        val[i] = __dadd_rn(__dmul_rn((double)((packed >> (4 * i)) & 0xF), __ldg(scales + g)), __ldg(zeros + g));
      }
    }
    if (kBf16) {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + e0;
      if (e0 + 7 < n) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 p = __floats2bfloat162_rn((float)val[2 * i], (float)val[2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&p);
        }
        *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        for (int i = 0; i < 8 && e0 + i < n; ++i) o[i] = __float2bfloat16_rn((float)val[i]);
      }
    } else {
      double* o = reinterpret_cast<double*>(out) + e0;
      for (int i = 0; i < 8; ++i)
        if (e0 + i < n) o[i] = val[i];
    }
  }
}

// Fast path (group_size % 32 == 0, n % 32 == 0, 16-byte aligned codes): a
// thread expands 16 packed bytes (32 elements of one group) per step — one
// 16-byte load, one scale/zero pair, 4 x 16-byte bf16 stores (or 16 x 16-byte
// fp64 stores) — with two steps in flight, so the kernel streams at HBM rate
// instead of issuing 4-byte loads one at a time.
template <bool kBf16>
__global__ void __launch_bounds__(kThreads) dequant32_kernel(const uint4* __restrict__ codes,
                                                             const double* __restrict__ scales,
                                                             const double* __restrict__ zeros, int64_t group_size,
                                                             int64_t n32, void* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t v0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; v0 < n32; v0 += 2 * stride) {
    uint4 pk[2];
    double sc[2], zp[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t v = v0 + u * stride;
      if (v < n32) {
        pk[u] = __ldcs(codes + v);
        const int64_t g = v * 32 / group_size;
        sc[u] = __ldg(scales + g);
        zp[u] = __ldg(zeros + g);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= n32) break;
      const uint32_t words[4] = {pk[u].x, pk[u].y, pk[u].z, pk[u].w};
#pragma unroll
      for (int wq = 0; wq < 4; ++wq) {
        double val[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          val[i] = __dadd_rn(__dmul_rn((double)((words[wq] >> (4 * i)) & 0xF), sc[u]), zp[u]);
        if (kBf16) {
          uint32_t w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 p2 = __floats2bfloat162_rn((float)val[2 * i], (float)val[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&p2);
          }
          __stcs(reinterpret_cast<uint4*>(out) + v * 4 + wq, make_uint4(w[0], w[1], w[2], w[3]));
        } else {
          double2* o = reinterpret_cast<double2*>(out) + (v * 32 + wq * 8) / 2;
#pragma unroll
          for (int i = 0; i < 4; ++i) __stcs(o + i, make_double2(val[2 * i], val[2 * i + 1]));
        }
      }
    }
  }
}

}  // namespace quant
}  // namespace hap

extern "C" int hap_int4_dequant(const uint8_t* codes, const double* scales, const double* zero_points,
                                int64_t group_size, int64_t n, void* out, int32_t out_bf16, void* stream) {
  using namespace hap::quant;
  if (!codes || !scales || !zero_points || !out || group_size < 1 || n < 0) return HAP_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(codes) & 3) || (reinterpret_cast<uintptr_t>(out) & 15)) return HAP_ERR_MISALIGNED;
  if (n == 0) return HAP_OK;
  if (group_size % 32 == 0 && n % 32 == 0 && (reinterpret_cast<uintptr_t>(codes) & 15) == 0) {
    const int64_t n32 = n / 32;
    int64_t g32 = (n32 + 2 * kThreads - 1) / (2 * kThreads);
    if (g32 > 148 * 16) g32 = 148 * 16;
    cudaStream_t st32 = reinterpret_cast<cudaStream_t>(stream);
    const uint4* c4 = reinterpret_cast<const uint4*>(codes);
    if (out_bf16)
      { if (hap::launch_k(dequant32_kernel<true>, dim3((int)g32), dim3(kThreads), 0, st32, c4, scales, zero_points, group_size, n32, out) != cudaSuccess) return HAP_ERR_LAUNCH; }
    else
      { if (hap::launch_k(dequant32_kernel<false>, dim3((int)g32), dim3(kThreads), 0, st32, c4, scales, zero_points, group_size, n32, out) != cudaSuccess) return HAP_ERR_LAUNCH; }
    HAP_CHECK_LAUNCH();
    return HAP_OK;
  }
  const int64_t n8 = (n + 7) / 8;
  int64_t grid = (n8 + kThreads - 1) / kThreads;
  if (grid > 148 * 32) grid = 148 * 32;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (out_bf16)
    { if (hap::launch_k(dequant_kernel<true>, dim3((int)grid), dim3(kThreads), 0, st, codes, scales, zero_points, group_size, n, out) != cudaSuccess) return HAP_ERR_LAUNCH; }
  else
    { if (hap::launch_k(dequant_kernel<false>, dim3((int)grid), dim3(kThreads), 0, st, codes, scales, zero_points, group_size, n, out) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
