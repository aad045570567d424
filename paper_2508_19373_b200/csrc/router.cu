// Gating: router logits (fp32, fixed sequential reduction order), softmax,
// top-k with lower-index tie break, optional renormalisation, optional
// Qwen-style shared-expert sigmoid gate.
//
// Layout: one lane owns one token; a warp covers 32 tokens.  The router weight
// is staged in shared memory transposed to [h/8][NE][8] so that, for a given
// 8-element slice of h, every lane reads the same 16-byte vector per expert
// (smem broadcast, conflict-free).  Each lane accumulates
//     acc[e] = fma(x[t,j], w[e,j], acc[e])   for j = 0 .. h-1 in order,
// which equals the sequential fp32 sum of exact bf16*bf16 products — the
// order the CPU oracle (oracle/moe_block.py:router_logits) reproduces bit for
// bit, so the top-k indices are bit-exact against it.
//
// Models: router term 2*T*h*E of expert_flops (reference arch.py:177); HF
// semantics of MixtralTopKRouter / Qwen2MoeTopKRouter (softmax -> top-k ->
// optional renorm).
#include "common.cuh"

namespace hap {
namespace router {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kSmemBudget = 96 * 1024;

template <int NE>
__global__ void __launch_bounds__(kThreads) router_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ w, int T, int h,
                                                          int n_rows_w, int E, int top_k, int renorm,
                                                          int has_shared, int chunk, int32_t* __restrict__ topk_idx,
                                                          float* __restrict__ topk_w, float* __restrict__ shared_gate,
                                                          float* __restrict__ logits_out) {
  extern __shared__ uint4 wsm[];  // [chunk/8][NE] uint4 (8 bf16 each)
  const int t = blockIdx.x * kThreads + threadIdx.x;
  const bool valid = t < T;
  const __nv_bfloat16* xrow = x + (int64_t)(valid ? t : 0) * h;

  float acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.f;

  for (int c0 = 0; c0 < h; c0 += chunk) {
    const int clen = min(chunk, h - c0);
    __syncthreads();
    // stage w[:, c0:c0+clen] transposed into [clen/8][NE]
    const int nvec = (clen / 8) * NE;
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      const int e = i % NE;
      const int j8 = i / NE;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (e < n_rows_w) v = *reinterpret_cast<const uint4*>(w + (int64_t)e * h + c0 + j8 * 8);
      wsm[i] = v;
    }
    __syncthreads();
    for (int j8 = 0; j8 < clen / 8; ++j8) {
      const uint4 xv = *reinterpret_cast<const uint4*>(xrow + c0 + j8 * 8);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      float xf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(xw[i]);
        xf[2 * i] = f.x;
        xf[2 * i + 1] = f.y;
      }
      const uint4* wrow = wsm + j8 * NE;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const uint4 wv = wrow[e];
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = unpack_bf16x2(ww[i]);
          acc[e] = __fmaf_rn(xf[2 * i], f.x, acc[e]);
          acc[e] = __fmaf_rn(xf[2 * i + 1], f.y, acc[e]);
        }
      }
    }
  }
  if (!valid) return;

  if (logits_out) {
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e < E) logits_out[(int64_t)t * E + e] = acc[e];
  }
  // softmax denominator over the E routed experts (fp32)
  float mx = -INFINITY;
#pragma unroll
  for (int e = 0; e < NE; ++e)
    if (e < E) mx = fmaxf(mx, acc[e]);
  float denom = 0.f;
#pragma unroll
  for (int e = 0; e < NE; ++e)
    if (e < E) denom += expf(acc[e] - mx);

  // top-k on logits; strict '>' keeps the lowest index on ties
  uint32_t taken[(NE + 31) / 32];
#pragma unroll
  for (int i = 0; i < (NE + 31) / 32; ++i) taken[i] = 0;
  float sel_w[32];
  int sel_i[32];
  float wsum = 0.f;
  for (int s = 0; s < top_k; ++s) {
    float best = -INFINITY;
    int bi = -1;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool free_e = e < E && !((taken[e >> 5] >> (e & 31)) & 1u);
      if (free_e && (bi < 0 || acc[e] > best)) {
        best = acc[e];
        bi = e;
      }
    }
    taken[bi >> 5] |= 1u << (bi & 31);
    const float p = expf(best - mx) / denom;
    sel_w[s] = p;
    sel_i[s] = bi;
    wsum += p;
  }
  for (int s = 0; s < top_k; ++s) {
    topk_idx[(int64_t)t * top_k + s] = sel_i[s];
    topk_w[(int64_t)t * top_k + s] = renorm ? sel_w[s] / wsum : sel_w[s];
  }
  if (has_shared && shared_gate) {
    float g = 0.f;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e == E) g = acc[e];
    shared_gate[t] = 1.f / (1.f + expf(-g));
  }
}

template <int NE>
static int launch(const void* x, int64_t T, int64_t h, const void* w, int64_t E, int64_t k, int renorm,
                  int has_shared, int32_t* idx, float* tw, float* sg, float* logits, cudaStream_t st) {
  int chunk = (kSmemBudget / (NE * 2)) / 256 * 256;
  if (chunk > h) chunk = (int)h;
  if (chunk < 256) chunk = 256;
  const int smem = (chunk / 8) * NE * 16;
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)router_kernel<NE>, kSmemBudget)) return HAP_ERR_LAUNCH;
    configured = 1;
  }
  const int grid = (int)((T + kThreads - 1) / kThreads);
  router_kernel<NE><<<grid, kThreads, smem, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w), (int)T, (int)h,
      (int)(E + has_shared), (int)E, (int)k, renorm, has_shared, chunk, idx, tw, sg, logits);
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace router
}  // namespace hap

extern "C" int hap_router_topk(const void* x, int64_t T, int64_t h, const void* w, int64_t n_experts,
                               int64_t top_k, int32_t renormalize, int32_t has_shared_gate, int32_t* topk_idx,
                               float* topk_w, float* shared_gate, float* logits_out, void* stream) {
  using namespace hap::router;
  if (!x || !w || !topk_idx || !topk_w || T < 0 || h <= 0) return HAP_ERR_INVALID_ARG;
  if (n_experts < 1 || top_k < 1 || top_k > n_experts || top_k > 32) return HAP_ERR_INVALID_ARG;
  if (has_shared_gate && !shared_gate) return HAP_ERR_INVALID_ARG;
  if (h % 256) return HAP_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) return HAP_ERR_MISALIGNED;
  if (T == 0) return HAP_OK;
  const int64_t rows = n_experts + (has_shared_gate ? 1 : 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int hs = has_shared_gate ? 1 : 0;
#define HAP_ROUTER_CASE(NE) \
  if (rows <= NE) return launch<NE>(x, T, h, w, n_experts, top_k, renormalize, hs, topk_idx, topk_w, shared_gate, logits_out, st);
  HAP_ROUTER_CASE(8)
  HAP_ROUTER_CASE(16)
  HAP_ROUTER_CASE(32)
  HAP_ROUTER_CASE(64)
  HAP_ROUTER_CASE(72)
#undef HAP_ROUTER_CASE
  return HAP_ERR_UNSUPPORTED;
}
