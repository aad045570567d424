// Gating: router logits (fp32, fixed reduction order), softmax, top-k with
// lower-index tie break, optional renormalisation, optional Qwen-style
// shared-expert sigmoid gate.
//
// Layout: a CTA covers 32 tokens (one per lane) with 8 warps; warp p owns the
// contiguous h-range [p*h/8, (p+1)*h/8).  Each lane accumulates, for every
// expert e, the sequential fp32 chain
//     part_p[e] = fma(x[t,j], w[e,j], part_p[e])   j over range p in order
// (bf16*bf16 products are exact in fp32, so this is the sequential fp32 sum
// of products), and the 8 partials are then added in order p = 0..7.  The
// CPU oracle (oracle/moe_block.py:router_logits) reproduces exactly this
// order, so the logits — and hence the top-k indices — are bit-exact.
// x rows are prefetched 4 x 16 B ahead per lane; router rows are read as
// warp-broadcast 16-byte loads that stay resident in L1.
//
// Models: router term 2*T*h*E of expert_flops (reference arch.py:177); HF
// semantics of MixtralTopKRouter / Qwen2MoeTopKRouter (softmax -> top-k ->
// optional renorm).
#include <cstdlib>

#include "common.cuh"

namespace hap {
namespace router {

constexpr int kRanges = 8;              // == warps per CTA; fixed by the parity contract
constexpr int kThreads = kRanges * 32;
constexpr int kPrefetch = 4;
constexpr int kSmallPrefetch = 16;  // router rows stream from L2: 16 x 16 B in flight per thread
constexpr int kSmallT = 1024;         // <= this many tokens: one CTA per token

// Softmax over the E routed logits, top-k on logits (strict '>' keeps the lower
// index on ties), optional renormalisation, shared-expert sigmoid gate.
template <int NE>
__device__ __forceinline__ void finish_token(const float (&acc)[NE], int t, int E, int top_k, int renorm,
                                             int has_shared, int32_t* __restrict__ topk_idx,
                                             float* __restrict__ topk_w, float* __restrict__ shared_gate,
                                             float* __restrict__ logits_out) {
  if (logits_out) {
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e < E) logits_out[(int64_t)t * E + e] = acc[e];
  }
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
    topk_idx[(int64_t)t * top_k + s] = bi;
    topk_w[(int64_t)t * top_k + s] = p;
    wsum += p;
  }
  if (renorm) {
    const float inv = 1.f / wsum;
    for (int s = 0; s < top_k; ++s) topk_w[(int64_t)t * top_k + s] *= inv;
  }
  if (has_shared && shared_gate) {
    float g = 0.f;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e == E) g = acc[e];
    shared_gate[t] = 1.f / (1.f + expf(-g));
  }
}

// Small-T variant (decode): one CTA per token; thread (p, e) runs exactly the
// sequential fma chain the large kernel's lane runs for (token, expert e,
// range p), so the logits are bit-identical between the two variants.
template <int NE, bool kStage>
__global__ void __launch_bounds__(kRanges * NE) router_small_kernel(const __nv_bfloat16* __restrict__ x,
                                                                    const __nv_bfloat16* __restrict__ w, int T,
                                                                    int h, int n_rows_w, int E, int top_k,
                                                                    int renorm, int has_shared,
                                                                    int32_t* __restrict__ topk_idx,
                                                                    float* __restrict__ topk_w,
                                                                    float* __restrict__ shared_gate,
                                                                    float* __restrict__ logits_out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ uint4 xs[];  // token row (h/8 vectors), then (kStage) the router rows
  __shared__ float part[kRanges][NE];
  __shared__ __align__(8) uint64_t bar;
  const int t = blockIdx.x;
  const uint4* xrow = reinterpret_cast<const uint4*>(x + (int64_t)t * h);
  const int p = threadIdx.x / NE, e = threadIdx.x % NE;
  const int hr = h / kRanges;
  const int nv = hr / 8;
  // kStage: the token row and every (router row, h-range) segment arrive by 1D
  // bulk copies in one round trip; segments sit nv+1 vectors apart so the 64
  // threads' reads fall in different banks.  (The streaming variant needs
  // ~4 dependent L2/DRAM round trips per thread: 15 us for Mixtral decode.)
  uint4* ws = xs + h / 8;
  if (kStage) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, (uint32_t)(h * 2) + (uint32_t)n_rows_w * (uint32_t)(h * 2));
      bulk_load(xs, xrow, (uint32_t)(h * 2), &bar);
      for (int r = 0; r < n_rows_w * kRanges; ++r)
        bulk_load(ws + r * (nv + 1), w + (int64_t)r * hr, (uint32_t)(hr * 2), &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int i = threadIdx.x; i < h / 8; i += blockDim.x) xs[i] = __ldg(xrow + i);
    __syncthreads();
  }
  float acc = 0.f;
  if (e < n_rows_w) {
    const uint4* xr = xs + p * nv;
    if (kStage) {
      const uint4* wr = ws + (e * kRanges + p) * (nv + 1);
#pragma unroll 4
      for (int v = 0; v < nv; ++v) {
        const uint4 wv = wr[v];
        const uint4 xv = xr[v];
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 fx = unpack_bf16x2(xw[q]);
          const float2 fw = unpack_bf16x2(ww[q]);
          acc = __fmaf_rn(fx.x, fw.x, acc);
          acc = __fmaf_rn(fx.y, fw.y, acc);
        }
      }
    } else {
      const uint4* wr = reinterpret_cast<const uint4*>(w + (int64_t)e * h + p * hr);
      uint4 wb[kSmallPrefetch];
#pragma unroll
      for (int i = 0; i < kSmallPrefetch; ++i) wb[i] = i < nv ? __ldg(wr + i) : make_uint4(0, 0, 0, 0);
      for (int v0 = 0; v0 < nv; v0 += kSmallPrefetch) {
#pragma unroll
        for (int i = 0; i < kSmallPrefetch; ++i) {
          const int v = v0 + i;
          if (v >= nv) break;
          const uint4 wv = wb[i];
          if (v + kSmallPrefetch < nv) wb[i] = __ldg(wr + v + kSmallPrefetch);
          const uint4 xv = xr[v];
          const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
          const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 fx = unpack_bf16x2(xw[q]);
            const float2 fw = unpack_bf16x2(ww[q]);
            acc = __fmaf_rn(fx.x, fw.x, acc);
            acc = __fmaf_rn(fx.y, fw.y, acc);
          }
        }
      }
    }
  }
  part[p][e] = acc;
  __syncthreads();
  if (threadIdx.x != 0) return;
  float tot[NE];
#pragma unroll
  for (int ee = 0; ee < NE; ++ee) {
    float s2 = part[0][ee];
#pragma unroll
    for (int pp = 1; pp < kRanges; ++pp) s2 = __fadd_rn(s2, part[pp][ee]);
    tot[ee] = s2;
  }
  finish_token<NE>(tot, t, E, top_k, renorm, has_shared, topk_idx, topk_w, shared_gate, logits_out);
}

// finish_token for one token by a whole warp (the wide router's last CTA):
// lane l holds logits l, l+32, l+64; the max, the softmax denominator and each
// of the top_k arg-max rounds are warp reductions (ties -> lower index, as in
// finish_token) instead of one thread's sequential passes over ~65 logits.
__device__ __forceinline__ void finish_token_warp(const float* __restrict__ lg, int n_rows, int t, int E, int top_k,
                                                  int renorm, int has_shared, int32_t* __restrict__ topk_idx,
                                                  float* __restrict__ topk_w, float* __restrict__ shared_gate,
                                                  float* __restrict__ logits_out) {
  const int lane = threadIdx.x & 31;
  float v[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < n_rows ? __ldcg(lg + e) : 0.f;
    if (logits_out && e < E) logits_out[(int64_t)t * E + e] = v[i];
  }
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (lane + 32 * i < E) mx = fmaxf(mx, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float den = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (lane + 32 * i < E) den += expf(v[i] - mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  bool taken[3] = {false, false, false};
  float wsum = 0.f;
  for (int s = 0; s < top_k; ++s) {
    float best = -INFINITY;
    int bi = INT32_MAX;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int e = lane + 32 * i;
      if (e < E && !taken[i] && (bi == INT32_MAX || v[i] > best)) {
        best = v[i];
        bi = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi != INT32_MAX && (bi == INT32_MAX || ob > best || (ob == best && oi < bi))) {
        best = ob;
        bi = oi;
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (bi == lane + 32 * i) taken[i] = true;
    const float p = expf(best - mx) / den;
    wsum += p;
    if (lane == 0) {
      topk_idx[(int64_t)t * top_k + s] = bi;
      topk_w[(int64_t)t * top_k + s] = p;
    }
  }
  if (lane == 0) {
    if (renorm) {
      const float inv = 1.f / wsum;
      for (int s = 0; s < top_k; ++s) topk_w[(int64_t)t * top_k + s] *= inv;
    }
    if (has_shared && shared_gate) shared_gate[t] = 1.f / (1.f + expf(-__ldcg(lg + E)));
  }
}

// Small T, wide router (rows > 8): one CTA per (token, group of 8 router rows)
// instead of one per token, so a decode step with few tokens streams the
// router rows on rows/8 SMs.  Chains and range order are those of
// router_small_kernel (bit-identical logits); each CTA parks its 8 logits in a
// scratch row of the caller's workspace, and the token's last CTA (atomic
// count, reset by itself) runs the softmax / top-k.  Workspace layout
// (independent of T, so launches of any size can share it): int32
// cnt[kSmallT] (zero before the first launch; every launch leaves it zeroed),
// then float logits[T][kMaxRouterRows].  Concurrent launches need distinct
// workspaces.
constexpr int kGroupRows = 8;
constexpr int kGroupTB = 8;        // tokens per CTA of the blocked wide router
constexpr int kGroupTBMinT = 32;   // ... from this many tokens on (16: 9.8 -> 13.6 us)
constexpr int kMaxRouterRows = 80;
constexpr int64_t kGroupCntBytes = (int64_t)kSmallT * 4;

// TB > 1: one CTA per (block of TB tokens, group of G router rows), warp w
// taking token w of the block with the same (row, range) thread layout, so the
// G router rows staged in shared memory serve TB tokens (mid-size decode
// batches: Qwen2-57B T = 512 had 8704 one-warp CTAs each re-staging its rows;
// kRanges * G threads per token, the first warp of each finishes it).
// The block's last CTA finishes its TB tokens, one warp each; the block counter
// is the workspace slot of its first token.
template <int NE, int G, int TB>
__global__ void __launch_bounds__(kRanges * G * TB) router_group_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w, int T, int h, int n_rows_w, int E,
    int top_k, int renorm, int has_shared, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
    float* __restrict__ shared_gate, float* __restrict__ logits_out, uint8_t* __restrict__ scratch) {
  constexpr int kPer = kRanges * G;  // threads per token (a whole number of warps)
  static_assert(kPer % 32 == 0, "kRanges * G must be a multiple of the warp size");
  pdl_trigger();
  pdl_wait();
  int* cnt_ws = reinterpret_cast<int*>(scratch);
  float* logits_ws = reinterpret_cast<float*>(scratch + kGroupCntBytes);
  extern __shared__ uint4 xs[];  // TB token rows (h/8 vectors each), then the group's (row, range) segments
  __shared__ float part[TB][kRanges][G];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int last_s;
  const int t0 = blockIdx.x * TB, g = blockIdx.y, n_groups = gridDim.y;
  const int tb = threadIdx.x / kPer, lt = threadIdx.x % kPer;
  const int p = lt / G, el = lt % G, e = g * G + el;
  const int t = t0 + tb;
  const int n_tok = min(TB, T - t0);
  const int hr = h / kRanges, nv = hr / 8;
  const int rows_here = min(G, n_rows_w - g * G);
  // token rows and this group's router rows arrive by 1D bulk copies in one
  // round trip; segments nv+1 vectors apart keep the threads' reads in
  // different banks
  uint4* ws = xs + TB * (h / 8);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(h * 2) * (uint32_t)(n_tok + rows_here));
    for (int i = 0; i < n_tok; ++i)
      bulk_load(xs + i * (h / 8), x + (int64_t)(t0 + i) * h, (uint32_t)(h * 2), &bar);
    for (int r = 0; r < rows_here * kRanges; ++r) {
      const int rl = r / kRanges, pp = r % kRanges;
      bulk_load(ws + (rl * kRanges + pp) * (nv + 1), w + (int64_t)(g * G + rl) * h + pp * hr,
                (uint32_t)(hr * 2), &bar);
    }
  }
  mbar_wait(&bar, 0);
  float acc = 0.f;
  if (e < n_rows_w && tb < n_tok) {
    const uint4* wr = ws + (el * kRanges + p) * (nv + 1);
    const uint4* xr = xs + tb * (h / 8) + p * nv;
#pragma unroll 4
    for (int v = 0; v < nv; ++v) {
      const uint4 wv = wr[v];
      const uint4 xv = xr[v];
      const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 fx = unpack_bf16x2(xw[q]);
        const float2 fw = unpack_bf16x2(ww[q]);
        acc = __fmaf_rn(fx.x, fw.x, acc);
        acc = __fmaf_rn(fx.y, fw.y, acc);
      }
    }
  }
  part[tb][p][el] = acc;
  __syncthreads();
  if (lt < G && e < n_rows_w && tb < n_tok) {
    float s2 = part[tb][0][el];
#pragma unroll
    for (int pp = 1; pp < kRanges; ++pp) s2 = __fadd_rn(s2, part[tb][pp][el]);
    logits_ws[(int64_t)t * kMaxRouterRows + e] = s2;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_s = atomicAdd(&cnt_ws[t0], 1) == n_groups - 1;
  __syncthreads();
  if (!last_s || tb >= n_tok || lt >= 32) return;
  __threadfence();
  if (threadIdx.x == 0) cnt_ws[t0] = 0;  // ready for the next launch
  finish_token_warp(logits_ws + (int64_t)t * kMaxRouterRows, n_rows_w, t, E, top_k, renorm, has_shared, topk_idx,
                    topk_w, shared_gate, logits_out);
}

template <int NE>
__global__ void __launch_bounds__(kThreads) router_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ w, int T, int h,
                                                          int n_rows_w, int E, int top_k, int renorm,
                                                          int has_shared, int32_t* __restrict__ topk_idx,
                                                          float* __restrict__ topk_w, float* __restrict__ shared_gate,
                                                          float* __restrict__ logits_out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float part[];  // [kRanges][NE][33]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 32 + lane;
  const bool valid = t < T;
  const int hr = h / kRanges;
  const int j0 = warp * hr;
  const uint4* xrow = reinterpret_cast<const uint4*>(x + (int64_t)(valid ? t : 0) * h + j0);
  const int nv = hr / 8;

  float acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.f;

  uint4 xb[kPrefetch];
#pragma unroll
  for (int i = 0; i < kPrefetch; ++i) xb[i] = i < nv ? __ldg(xrow + i) : make_uint4(0, 0, 0, 0);

  for (int v0 = 0; v0 < nv; v0 += kPrefetch) {
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i) {
      const int v = v0 + i;
      if (v >= nv) break;
      const uint4 xv = xb[i];
      if (v + kPrefetch < nv) xb[i] = __ldg(xrow + v + kPrefetch);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      float xf[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack_bf16x2(xw[q]);
        xf[2 * q] = f.x;
        xf[2 * q + 1] = f.y;
      }
      const int j = j0 + v * 8;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        if (e < n_rows_w) {
          const uint4 wv = __ldg(reinterpret_cast<const uint4*>(w + (int64_t)e * h + j));
          const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = unpack_bf16x2(ww[q]);
            acc[e] = __fmaf_rn(xf[2 * q], f.x, acc[e]);
            acc[e] = __fmaf_rn(xf[2 * q + 1], f.y, acc[e]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) part[(warp * NE + e) * 33 + lane] = acc[e];
  __syncthreads();
  if (warp != 0 || !valid) return;

  // fixed-order sum of the range partials: ((p0 + p1) + p2) + ...
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    float s = part[e * 33 + lane];
#pragma unroll
    for (int p = 1; p < kRanges; ++p) s = __fadd_rn(s, part[(p * NE + e) * 33 + lane]);
    acc[e] = s;
  }

  finish_token<NE>(acc, t, E, top_k, renorm, has_shared, topk_idx, topk_w, shared_gate, logits_out);
}

// Large-T variant: CTA = 32*TPL tokens x 8 h-ranges, lane owns tokens
// (t0 + lane [, t0 + lane + 32]) of its warp's range.  Each warp streams its
// range in CH-element chunks through a 2-stage TMA ring: the token rows
// (CH x 32*TPL box, swizzled) and the router rows of that chunk (CH x NE box,
// bf16, OOB rows zero-filled) land on one barrier per stage.  Each warp then
// re-expands its router chunk to fp32 transposed to [j][e], so one broadcast
// 16-byte load yields the weights of experts e..e+3 at element j, and the
// chains (token, e) and (token, e+1) advance together in one packed FFMA2
// (fma.rn.f32x2: two independent fma.rn.f32, rounding unchanged).  Every
// (token, expert, range) chain and the ordered sum of the range partials are
// exactly those of router_kernel: logits are bit-identical.
constexpr int kXStages = 2;


template <int NE, int TPL, int CH>
struct RouterTmaGeo {
  static_assert(NE % 4 == 0, "expert quads");
  static constexpr int kTB = 32 * TPL;                       // tokens per CTA
  static constexpr int kXBytes = kTB * CH * 2;               // token box per warp-stage
  static constexpr int kWBytes = NE * CH * 2;                // router box per warp-stage
  static constexpr int kStageBytes = kXBytes + kWBytes;
  static constexpr int kWT = CH * NE * 4;                    // fp32 [j][e] router chunk per warp
  static constexpr int kRing = kRanges * (kXStages * kStageBytes + kWT);
  static constexpr int kPart = kRanges * NE * (kTB + 1) * 4;  // partial table (overlays the rings)
  static constexpr int kSmem = (kRing > kPart ? kRing : kPart) + 1024;
};

template <int NE, int TPL, int CH>
__global__ void __launch_bounds__(kThreads, NE <= 8 ? (TPL == 1 ? 4 : 2) : 1)
    router_tma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int T,
                      int h, int E, int top_k, int renorm, int has_shared, int32_t* __restrict__ topk_idx,
                      float* __restrict__ topk_w, float* __restrict__ shared_gate, float* __restrict__ logits_out) {
  pdl_trigger();
  pdl_wait();
  using G = RouterTmaGeo<NE, TPL, CH>;
  constexpr int kTB = G::kTB;
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = smem_align1024(dsm_raw);
  __shared__ __align__(8) uint64_t bars[kRanges][kXStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = dsm + warp * (kXStages * G::kStageBytes + G::kWT);
  float* wT = reinterpret_cast<float*>(ring + kXStages * G::kStageBytes);  // [CH][NE]
  uint64_t* bar = bars[warp];
  const int tb0 = blockIdx.x * kTB;
  const int hr = h / kRanges, j0 = warp * hr, nch = hr / CH;
  if (lane == 0) {
    for (int s2 = 0; s2 < kXStages; ++s2) mbar_init(&bar[s2], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto issue = [&](int c, int stage) {
    if (lane == 0) {
      uint8_t* st = ring + stage * G::kStageBytes;
      mbar_arrive_expect_tx(&bar[stage], G::kStageBytes);
      tma_load_2d(st, &tmX, &bar[stage], j0 + c * CH, tb0, kEvictFirst);
      tma_load_2d(st + G::kXBytes, &tmW, &bar[stage], j0 + c * CH, 0, kEvictLast);
    }
  };
  for (int c = 0; c < kXStages && c < nch; ++c) issue(c, c);

  uint64_t acc2[TPL][NE / 2];  // chains (token i, e) and (token i, e+1) as one fp32 pair
#pragma unroll
  for (int i = 0; i < TPL; ++i)
#pragma unroll
    for (int e = 0; e < NE / 2; ++e) acc2[i][e] = 0ull;
  // swizzle phase of rows lane and lane + 32: 16-byte chunk c of row r sits at
  // c ^ (r & 7) (128B rows) or c ^ ((r >> 1) & 3) (64B rows)
  const int sw = CH == 64 ? (lane & 7) : ((lane >> 1) & 3);
  for (int c = 0; c < nch; ++c) {
    const int stage = c % kXStages;
    mbar_wait(&bar[stage], (c / kXStages) & 1);
    const uint8_t* xst = ring + stage * G::kStageBytes;
    const uint4* wst = reinterpret_cast<const uint4*>(xst + G::kXBytes);  // [NE][CH/8] 16-byte vectors
#pragma unroll
    for (int it = lane; it < NE * CH / 8; it += 32) {
      const int e = it / (CH / 8), v = it % (CH / 8);
      const uint4 wv = wst[it];
      const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack_bf16x2(ww[q]);
        wT[(8 * v + 2 * q) * NE + e] = f.x;
        wT[(8 * v + 2 * q + 1) * NE + e] = f.y;
      }
    }
    __syncwarp();
#pragma unroll 2
    for (int v = 0; v < CH / 8; ++v) {
      float xf[TPL][8];
#pragma unroll
      for (int i = 0; i < TPL; ++i) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xst + (lane + 32 * i) * (CH * 2) + ((v ^ sw) << 4));
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = unpack_bf16x2(xw[q]);
          xf[i][2 * q] = f.x;
          xf[i][2 * q + 1] = f.y;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint64_t xd[TPL];
#pragma unroll
        for (int i = 0; i < TPL; ++i) xd[i] = f2dup(xf[i][q]);
        const ulonglong2* wrow = reinterpret_cast<const ulonglong2*>(wT + (8 * v + q) * NE);
#pragma unroll
        for (int e4 = 0; e4 < NE / 4; ++e4) {
          const ulonglong2 w4 = wrow[e4];  // same address in every lane: broadcast
#pragma unroll
          for (int i = 0; i < TPL; ++i) {
            ffma2(acc2[i][2 * e4], xd[i], w4.x);
            ffma2(acc2[i][2 * e4 + 1], xd[i], w4.y);
          }
        }
      }
    }
    __syncwarp();  // stage and router chunk consumed by every lane
    if (c + kXStages < nch) issue(c + kXStages, stage);
  }
  __syncthreads();  // the partial table below overlays other warps' stages
  float* part = reinterpret_cast<float*>(dsm);  // [kRanges][NE][kTB + 1]
#pragma unroll
  for (int i = 0; i < TPL; ++i)
#pragma unroll
    for (int e2 = 0; e2 < NE / 2; ++e2) {
      const float2 f = f2split(acc2[i][e2]);
      part[(warp * NE + 2 * e2) * (kTB + 1) + lane + 32 * i] = f.x;
      part[(warp * NE + 2 * e2 + 1) * (kTB + 1) + lane + 32 * i] = f.y;
    }
  __syncthreads();
  if (threadIdx.x >= kTB) return;
  const int tl = threadIdx.x, t = tb0 + tl;
  if (t >= T) return;
  float tot[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    float s2 = part[e * (kTB + 1) + tl];
#pragma unroll
    for (int pp = 1; pp < kRanges; ++pp) s2 = __fadd_rn(s2, part[(pp * NE + e) * (kTB + 1) + tl]);
    tot[e] = s2;
  }
  finish_token<NE>(tot, t, E, top_k, renorm, has_shared, topk_idx, topk_w, shared_gate, logits_out);
}

template <int NE, int TPL, int CH>
static int launch_router_tma(const void* x, int64_t T, int64_t h, const void* w, int64_t E, int has_shared,
                             int64_t k, int renorm, int32_t* idx, float* tw, float* sg, float* logits,
                             cudaStream_t st) {
  using G = RouterTmaGeo<NE, TPL, CH>;
  static_assert(G::kSmem <= 227 * 1024, "router smem");
  auto kern = router_tma_kernel<NE, TPL, CH>;
  static int configured_tma = 0;
  if (!configured_tma) {
    if (configure_smem((const void*)kern, G::kSmem)) return HAP_ERR_LAUNCH;
    configured_tma = 1;
  }
  CUtensorMap tmX, tmW;
  if (!encode_tmap_2d_bf16_sw(&tmX, x, (uint64_t)h, (uint64_t)T, (uint64_t)h * 2, CH, G::kTB, CH * 2) ||
      !encode_tmap_2d_bf16_sw(&tmW, w, (uint64_t)h, (uint64_t)(E + has_shared), (uint64_t)h * 2, CH, NE, 0))
    return HAP_ERR_DRIVER;
  if (hap::launch_k(kern, dim3((unsigned)((T + G::kTB - 1) / G::kTB)), dim3(kThreads), G::kSmem, st, tmX, tmW,
                    (int)T, (int)h, (int)E, (int)k, renorm, has_shared, idx, tw, sg, logits) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

template <int NE>
static int launch(const void* x, int64_t T, int64_t h, const void* w, int64_t E, int64_t k, int renorm,
                  int has_shared, int32_t* idx, float* tw, float* sg, float* logits, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  const int smem = kRanges * NE * 33 * (int)sizeof(float);
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)router_kernel<NE>, smem)) return HAP_ERR_LAUNCH;
    configured = 1;
  }
  // wide routers (more rows than one group) leave the per-token kernels for
  // the TMA-staged token-block kernel above wide_max_t tokens (A/B switch
  // HAP_ROUTER_WIDE_MAXT; logits are bit-identical across the variants)
  static const int64_t wide_max_t = [] {
    const char* e = getenv("HAP_ROUTER_WIDE_MAXT");
    return e ? (int64_t)atoi(e) : (int64_t)kSmallT;
  }();
  const bool wide_to_tma = E + has_shared > kGroupRows && T > wide_max_t && h % (kRanges * 32) == 0;
  if (T <= kSmallT && !wide_to_tma) {
    const int xs_bytes = (int)(h / 8) * 16;
    const int ws_bytes = (int)((E + has_shared) * kRanges) * (int)(h / kRanges / 8 + 1) * 16;
    constexpr int kStageLimit = 200 * 1024;
    static int configured_small = 0;
    if (!configured_small) {
      if (configure_smem((const void*)router_small_kernel<NE, false>, 64 * 1024) ||
          configure_smem((const void*)router_small_kernel<NE, true>, kStageLimit))
        return HAP_ERR_LAUNCH;
      configured_small = 1;
    }
    if (xs_bytes > 64 * 1024) return HAP_ERR_UNSUPPORTED;
    static const bool allow_stage = [] {
      const char* e = getenv("HAP_ROUTER_STAGE");  // A/B experiments only
      return e ? atoi(e) != 0 : true;
    }();
    const bool stage = allow_stage && xs_bytes + ws_bytes <= kStageLimit && (reinterpret_cast<uintptr_t>(w) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const int gs_bytes = xs_bytes + kGroupRows * kRanges * (int)(h / kRanges / 8 + 1) * 16;
    if (!stage && E + has_shared > kGroupRows && E + has_shared <= kMaxRouterRows && gs_bytes <= kStageLimit &&
        ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(ws)) & 15) == 0 &&
        ws && ws_bytes >= (size_t)(kGroupCntBytes + T * kMaxRouterRows * 4)) {
      // router rows per CTA: 4 (default: twice the CTAs of 8, half the rows
      // each — Qwen2-57B decode router 12.0 -> 9.7 us per call in a graph) or
      // 8 (HAP_ROUTER_GROUP=8 A/B switch)
      static const int grp = [] {
        const char* e = getenv("HAP_ROUTER_GROUP");
        return e && atoi(e) == 8 ? 8 : 4;
      }();
      // token blocks of kGroupTB tokens per CTA from kGroupTBMinT tokens on
      // (HAP_ROUTER_TB=0 A/B switch keeps one token per CTA)
      static const bool tb_ok = [] {
        const char* e = getenv("HAP_ROUTER_TB");
        return !(e && e[0] == '0');
      }();
      const int gtb_bytes = kGroupTB * xs_bytes + 4 * kRanges * (int)(h / kRanges / 8 + 1) * 16;
      const bool blocked = tb_ok && grp == 4 && T >= kGroupTBMinT && gtb_bytes <= kStageLimit;
      auto gkern = blocked ? router_group_kernel<NE, 4, kGroupTB>
                           : (grp == 4 ? router_group_kernel<NE, 4, 1> : router_group_kernel<NE, kGroupRows, 1>);
      static int configured_group = 0;
      if (!configured_group) {
        if (configure_smem((const void*)router_group_kernel<NE, 4, 1>, kStageLimit) ||
            configure_smem((const void*)router_group_kernel<NE, 4, kGroupTB>, kStageLimit) ||
            configure_smem((const void*)router_group_kernel<NE, kGroupRows, 1>, kStageLimit))
          return HAP_ERR_LAUNCH;
        configured_group = 1;
      }
      const int n_groups = (int)((E + has_shared + grp - 1) / grp);
      const int tb = blocked ? kGroupTB : 1;
      { if (hap::launch_kr(T, gkern, dim3((unsigned)((T + tb - 1) / tb), (unsigned)n_groups), dim3(kRanges * grp * tb),
                          blocked ? gtb_bytes : gs_bytes, st, reinterpret_cast<const __nv_bfloat16*>(x),
                          reinterpret_cast<const __nv_bfloat16*>(w), (int)T, (int)h, (int)(E + has_shared), (int)E,
                          (int)k, renorm, has_shared, idx, tw, sg, logits,
                          reinterpret_cast<uint8_t*>(ws)) != cudaSuccess) return HAP_ERR_LAUNCH; }
      HAP_CHECK_LAUNCH();
      return HAP_OK;
    }
    auto kern = stage ? router_small_kernel<NE, true> : router_small_kernel<NE, false>;
    { if (hap::launch_kr(T, kern, dim3((int)T), dim3(kRanges * NE), stage ? xs_bytes + ws_bytes : xs_bytes, st,
        reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w), (int)T, (int)h,
        (int)(E + has_shared), (int)E, (int)k, renorm, has_shared, idx, tw, sg, logits) != cudaSuccess) return HAP_ERR_LAUNCH; }
    HAP_CHECK_LAUNCH();
    return HAP_OK;
  }
  if (h % (kRanges * 32) == 0) {
    // TMA-staged variant, 32-element chunks, 2 tokens per lane (64-token CTAs,
    // 2 per SM).  1 token per lane (32-token CTAs, 4 per SM: twice the CTAs in
    // flight) measured slower, 59 vs 41 us at Mixtral prefill: the kernel is
    // issue-bound on the weight re-expansion and operand moves, which the
    // 2-token layout amortises over twice the tokens (HAP_ROUTER_TPL A/B switch)
    static const int tpl = [] {
      const char* e = getenv("HAP_ROUTER_TPL");
      return e ? atoi(e) : 2;
    }();
    if (NE <= 8 && tpl == 1)
      return launch_router_tma<NE, 1, 32>(x, T, h, w, E, has_shared, k, renorm, idx, tw, sg, logits, st);
    return launch_router_tma<NE, 2, 32>(x, T, h, w, E, has_shared, k, renorm, idx, tw, sg, logits, st);
  }
  const int grid = (int)((T + 31) / 32);
  { if (hap::launch_k(router_kernel<NE>, dim3(grid), dim3(kThreads), smem, st, 
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w), (int)T, (int)h,
      (int)(E + has_shared), (int)E, (int)k, renorm, has_shared, idx, tw, sg, logits) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace router
}  // namespace hap

extern "C" size_t hap_router_workspace_bytes(int64_t T, int64_t n_experts, int32_t has_shared_gate) {
  using namespace hap::router;
  if (T <= 0 || T > kSmallT || n_experts + (has_shared_gate ? 1 : 0) <= kGroupRows) return 0;
  return (size_t)(kGroupCntBytes + T * kMaxRouterRows * 4);
}

extern "C" int hap_router_topk(const void* x, int64_t T, int64_t h, const void* w, int64_t n_experts,
                               int64_t top_k, int32_t renormalize, int32_t has_shared_gate, int32_t* topk_idx,
                               float* topk_w, float* shared_gate, float* logits_out, void* workspace,
                               size_t ws_bytes, void* stream) {
  using namespace hap::router;
  if (!x || !w || !topk_idx || !topk_w || T < 0 || h <= 0) return HAP_ERR_INVALID_ARG;
  if (n_experts < 1 || top_k < 1 || top_k > n_experts || top_k > 32) return HAP_ERR_INVALID_ARG;
  if (has_shared_gate && !shared_gate) return HAP_ERR_INVALID_ARG;
  if (h % (8 * kRanges)) return HAP_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) return HAP_ERR_MISALIGNED;
  if (T == 0) return HAP_OK;
  const int64_t rows = n_experts + (has_shared_gate ? 1 : 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int hs = has_shared_gate ? 1 : 0;
#define HAP_ROUTER_CASE(NE) \
  if (rows <= NE) return launch<NE>(x, T, h, w, n_experts, top_k, renormalize, hs, topk_idx, topk_w, shared_gate, logits_out, workspace, ws_bytes, st);
  HAP_ROUTER_CASE(8)
  HAP_ROUTER_CASE(16)
  HAP_ROUTER_CASE(32)
  HAP_ROUTER_CASE(64)
  HAP_ROUTER_CASE(72)
#undef HAP_ROUTER_CASE
  return HAP_ERR_UNSUPPORTED;
}
