// Block glue: RMSNorm and rotary position embedding.
//
// Not modelled by the reference FLOP formulas (arch.py:145-178 has no
// norm/rope term); semantics follow the HF decoder layer the planner's
// ModelSpec presets describe (Mixtral / Qwen2-MoE RMSNorm with fp32
// statistics; rotate-half RoPE with inv_freq = theta^(-2i/d)).
#include "common.cuh"

namespace hap {
namespace norm {

constexpr int kThreads = 256;

// Store one 16-byte vector to out, or (dst_tab != nullptr) to every base in
// the device table — the all-gather push of hap_rmsnorm_multi: peer-mapped
// bases make the normalised rows leave over NVLink as they are produced.
__device__ __forceinline__ void store_row(uint4* out, const int64_t* __restrict__ dst_tab, int n_dst, int64_t off,
                                          uint4 v) {
  if (dst_tab == nullptr) {
    out[off] = v;
    return;
  }
  for (int d = 0; d < n_dst; ++d) reinterpret_cast<uint4*>(__ldg(dst_tab + d))[off] = v;
}

// One warp per row; the row is held in registers (h/256 16-byte vectors per lane).
template <int VPL>  // 16-byte vectors per lane
__global__ void __launch_bounds__(kThreads) rmsnorm_kernel(const uint4* __restrict__ x, int T, int hv, int ldxv,
                                                           const uint4* __restrict__ w, float eps,
                                                           uint4* __restrict__ out, int ldov,
                                                           const int64_t* __restrict__ dst_tab, int n_dst) {
  pdl_trigger();
  pdl_wait();
  const int row = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  uint4 v[VPL];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < hv ? __ldg(x + (int64_t)row * ldxv + c) : make_uint4(0, 0, 0, 0);
    const uint32_t u[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(u[j]);
      ss = fmaf(f.x, f.x, ss);
      ss = fmaf(f.y, f.y, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)(hv * 8) + eps);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c >= hv) break;
    const uint4 wv = __ldg(w + c);
    const uint32_t u[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
    const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(u[j]);
      const float2 g = unpack_bf16x2(ww[j]);
      o[j] = pack_bf16x2(f.x * inv * g.x, f.y * inv * g.y);
    }
    store_row(out, dst_tab, n_dst, (int64_t)row * ldov + c, make_uint4(o[0], o[1], o[2], o[3]));
  }
}

// Wide rows (h >= 2048): 128 threads per row, VPT 16-byte vectors per thread,
// fp32 sum of squares reduced warp-then-block in a fixed order.  ~40 registers,
// so 16 rows per SM are in flight (the warp-per-row kernel needs the whole row
// in a lane's registers and is latency-bound at 1 CTA per SM).
constexpr int kRowThreads = 128;
template <int VPT>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_row_kernel(const uint4* __restrict__ x, int T, int hv, int ldxv,
                                                                  const uint4* __restrict__ w, float eps,
                                                                  uint4* __restrict__ out, int ldov,
                                                                  const int64_t* __restrict__ dst_tab, int n_dst) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[kRowThreads / 32];
  const int row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = tid + kRowThreads * i;
    v[i] = c < hv ? __ldg(x + (int64_t)row * ldxv + c) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const uint32_t u[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(u[j]);
      ss = fmaf(f.x, f.x, ss);
      ss = fmaf(f.y, f.y, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float inv = rsqrtf(tot / (float)(hv * 8) + eps);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = tid + kRowThreads * i;
    if (c >= hv) break;
    const uint4 wv = __ldg(w + c);
    const uint32_t u[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
    const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(u[j]);
      const float2 g = unpack_bf16x2(ww[j]);
      o[j] = pack_bf16x2(f.x * inv * g.x, f.y * inv * g.y);
    }
    store_row(out, dst_tab, n_dst, (int64_t)row * ldov + c, make_uint4(o[0], o[1], o[2], o[3]));
  }
}

// One warp per (token, head) for the q and k heads; lane owns rotation pairs
// (i, i + d/2) for i = lane, lane + 32 (d = 128) or i = lane (d = 64).
__global__ void __launch_bounds__(kThreads) rope_kernel(__nv_bfloat16* __restrict__ qkv, int T, int64_t ld,
                                                        int n_heads_rot, int d, const int32_t* __restrict__ pos,
                                                        float theta) {
  pdl_trigger();
  pdl_wait();
  const int item = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (item >= T * n_heads_rot) return;
  const int t = item / n_heads_rot;
  const int hh = item % n_heads_rot;
  __nv_bfloat16* base = qkv + (int64_t)t * ld + (int64_t)hh * d;
  const int half = d / 2;
  const float p = (float)pos[t];
  for (int i = lane; i < half; i += 32) {
    // inv_freq computed exactly as HF: 1 / theta^((2i)/d) in fp32
    const float inv_freq = 1.0f / powf(theta, (float)(2 * i) / (float)d);
    const float ang = p * inv_freq;
    float s, c;
    sincosf(ang, &s, &c);
    const float x1 = __bfloat162float(base[i]);
    const float x2 = __bfloat162float(base[i + half]);
    base[i] = __float2bfloat16_rn(x1 * c - x2 * s);
    base[i + half] = __float2bfloat16_rn(x2 * c + x1 * s);
  }
}

}  // namespace norm
}  // namespace hap

using namespace hap::norm;

static int rmsnorm_launch(const void* x, int64_t T, int64_t h, int64_t ldx, const void* w, float eps, void* out,
                          int64_t ldo, const int64_t* dst_tab, int n_dst, void* stream) {
  if (!x || !w || (!out && !dst_tab) || T < 0 || h <= 0 || ldx < h || ldo < h) return HAP_ERR_INVALID_ARG;
  if (h % 8 || ldx % 8 || ldo % 8) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) & 15)
    return HAP_ERR_MISALIGNED;
  if (T == 0) return HAP_OK;
  const int hv = (int)(h / 8);
  const int vpl = (hv + 31) / 32;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (int)((T * 32 + kThreads - 1) / kThreads);
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* ov = reinterpret_cast<uint4*>(out);
  if (hv >= 2 * kRowThreads && hv <= 8 * kRowThreads) {
    const int vpt = (hv + kRowThreads - 1) / kRowThreads;
#define HAP_ROW_CASE(V)                                                                                          \
  if (vpt <= V) {                                                                                               \
    { if (hap::launch_kr(T, rmsnorm_row_kernel<V>, dim3((unsigned)T), dim3(kRowThreads), 0, st, xv, (int)T, hv,    \
                        (int)(ldx / 8), wv, eps, ov, (int)(ldo / 8), dst_tab, n_dst) != cudaSuccess)           \
        return HAP_ERR_LAUNCH; }                                                                                \
    HAP_CHECK_LAUNCH();                                                                                         \
    return HAP_OK;                                                                                              \
  }
    HAP_ROW_CASE(2)
    HAP_ROW_CASE(4)
    HAP_ROW_CASE(6)
    HAP_ROW_CASE(8)
#undef HAP_ROW_CASE
  }
#define HAP_NORM_CASE(V) \
  if (vpl <= V) { { if (hap::launch_kr(T, rmsnorm_kernel<V>, dim3(grid), dim3(kThreads), 0, st, xv, (int)T, hv, (int)(ldx / 8), wv, eps, ov, (int)(ldo / 8), dst_tab, n_dst) != cudaSuccess) return HAP_ERR_LAUNCH; } HAP_CHECK_LAUNCH(); return HAP_OK; }
  HAP_NORM_CASE(2)
  HAP_NORM_CASE(4)
  HAP_NORM_CASE(8)
  HAP_NORM_CASE(16)
  HAP_NORM_CASE(24)
  HAP_NORM_CASE(32)
#undef HAP_NORM_CASE
  return HAP_ERR_UNSUPPORTED;
}

extern "C" int hap_rmsnorm(const void* x, int64_t T, int64_t h, int64_t ldx, const void* w, float eps, void* out,
                           int64_t ldo, void* stream) {
  if (!out) return HAP_ERR_INVALID_ARG;
  return rmsnorm_launch(x, T, h, ldx, w, eps, out, ldo, nullptr, 0, stream);
}

extern "C" int hap_rmsnorm_multi(const void* x, int64_t T, int64_t h, int64_t ldx, const void* w, float eps,
                                 const int64_t* dst_tab, int32_t n_dst, int64_t ldo, void* stream) {
  if (!dst_tab || n_dst < 1 || n_dst > 64) return HAP_ERR_INVALID_ARG;
  return rmsnorm_launch(x, T, h, ldx, w, eps, nullptr, ldo, dst_tab, n_dst, stream);
}

extern "C" int hap_rope_qk(void* qkv, int64_t T, int64_t ld, int64_t n_q_heads, int64_t n_kv_heads,
                           int64_t head_dim, const int32_t* positions, float theta, void* stream) {
  if (!qkv || !positions || T < 0 || n_q_heads < 1 || n_kv_heads < 0 || head_dim < 2 || head_dim % 2)
    return HAP_ERR_INVALID_ARG;
  if (ld < (n_q_heads + n_kv_heads) * head_dim) return HAP_ERR_INVALID_ARG;
  if (T == 0) return HAP_OK;
  const int heads = (int)(n_q_heads + n_kv_heads);
  const int64_t items = T * heads;
  const int grid = (int)((items * 32 + kThreads - 1) / kThreads);
  { if (hap::launch_k(rope_kernel, dim3(grid), dim3(kThreads), 0, reinterpret_cast<cudaStream_t>(stream), 
      reinterpret_cast<__nv_bfloat16*>(qkv), (int)T, ld, heads, (int)head_dim, positions, theta) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
