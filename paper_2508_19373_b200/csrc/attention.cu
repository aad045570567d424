// Attention core entry points: causal GQA prefill (tcgen05 flash attention,
// attn_tc.cu) and split-KV GQA decode over a head-major KV cache.
//
// Decode: warp-pipelined split-KV (decode_mma_kernel below) writes fp32
// partial (o, m, l) per (sequence, query head, key split) and a merge kernel
// rescales the splits.  KV cache layout: [B, n_kv, max_len, d].
//
// Models: score+value term 4*n*kv_len*h of attention_flops (reference
// arch.py:161); decode kv_len = input_len + output_len//2 (planner.py:226).
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace hap {
int attn_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                    int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, int64_t head_dim, float scale,
                    int32_t causal, int* sched, cudaStream_t st);
size_t attn_prefill_tc_workspace_bytes();

namespace attn {


// ------------------------------------------------------------------ decode --
constexpr int kMaxG = 8;

// Cache row of key position k of (sequence b, kv head h).  Contiguous cache
// [B, n_kv, max_len, D]: (b*n_kv + h)*max_len + k.  Paged cache (block_table
// != nullptr): a pool of pages [n_pages, n_kv, page, D] and int32
// block_table[b][k / page] = page id (< 0: not allocated, returns -1); a
// 16-key decode chunk never crosses a page (page is a multiple of 16).
struct KvLayout {
  const int32_t* block_table;
  int max_pages, page;
};
__device__ __forceinline__ int64_t kv_row(const KvLayout& L, int b, int h, int n_kv, int max_len, int k) {
  if (L.block_table == nullptr) return ((int64_t)b * n_kv + h) * max_len + k;
  const int pg = L.block_table[(int64_t)b * L.max_pages + k / L.page];
  return pg < 0 ? -1 : ((int64_t)pg * n_kv + h) * L.page + k % L.page;
}

// Copy the new token's k and v (from the fused qkv row, after RoPE) into the cache.
template <int D>
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, int n_q, int n_kv,
                                 __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int max_len,
                                 const int32_t* __restrict__ pos, KvLayout L) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const int p = pos[b];
  if (p < 0 || p >= max_len) return;  // outside the cache: nothing is written
  if (kv_row(L, b, 0, n_kv, max_len, p) < 0) return;  // page not allocated
  const __nv_bfloat16* row = qkv + (int64_t)b * ld;
  for (int i = threadIdx.x; i < n_kv * D / 8; i += blockDim.x) {
    const int hh = i / (D / 8), c = (i % (D / 8)) * 8;
    const int64_t dst = kv_row(L, b, hh, n_kv, max_len, p) * D + c;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + hh) * D + c);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + n_kv + hh) * D + c);
  }
}

// Warp-pipelined decode (the production path).  Each warp is an independent
// worker over items (sequence, kv head, key split): a 3-stage ring of 16-key
// chunks of K and V arrives by TMA (2-D view of the cache, 128B swizzle), the
// G query heads of the group (rows of an m16 tile) meet the chunk through
// mma.sync m16n8k16 bf16 (S = Q K^T, then O += P V with P kept in registers),
// with an online base-2 softmax per row.  The item's (o, m, l) goes to the
// workspace for decode_merge_kernel.  Memory-level parallelism comes from
// 8 warps x 3 stages in flight per SM; the FLOPs are negligible.
constexpr int kDecWarps = 8;
constexpr int kDecStages = 3;
constexpr int kDecChunk = 16;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// byte offset of (row r, element e) in a [rows][64 bf16] tile written by TMA with SWIZZLE_128B
__device__ __forceinline__ uint32_t sw128(int r, int e) {
  return (uint32_t)(r * 128 + ((((e >> 3) ^ r) & 7) << 4) + ((e & 7) << 1));
}

struct DecItem {
  int b, kvh, k0, nk;
};

// Keys [0, min(pos[b] + 1, max_len)) of sequence b: a position outside the
// cache never makes the kernels touch memory beyond the sequence's rows
// (kv_append_kernel skips it; the host API rejects it where it can see it).
__device__ __forceinline__ DecItem dec_item(int item, int n_kv, int ns, int split, const int32_t* pos, int max_len) {
  DecItem it;
  const int bk = item / ns, s = item - bk * ns;
  it.b = bk / n_kv;
  it.kvh = bk - it.b * n_kv;
  it.k0 = s * split;
  it.nk = max(0, min(min(pos[it.b] + 1, max_len), it.k0 + split) - it.k0);
  return it;
}

template <int D, int G>
__global__ void __launch_bounds__(kDecWarps * 32, 1)
    decode_mma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __nv_bfloat16* __restrict__ qkv, int64_t ld, int max_len, const int32_t* __restrict__ pos,
                      int B, int n_q, int n_kv, float scale_log2, float* __restrict__ ws_o,
                      float* __restrict__ ws_ml, int ns, int split, KvLayout L) {
  pdl_trigger();
  pdl_wait();
  constexpr int H = D / 64;                        // 128-byte column halves of a row
  constexpr int kHalfBytes = kDecChunk * 128;      // 2 KB
  constexpr int kStageBytes = 2 * H * kHalfBytes;  // K + V of one chunk
  constexpr int NT = D / 8;                        // O n-tiles
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = smem_align1024(dsm_raw);
  __shared__ __align__(8) uint64_t bars[kDecWarps][kDecStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = dsm + warp * kDecStages * kStageBytes;
  uint64_t* full = bars[warp];
  if (lane == 0) {
    for (int s = 0; s < kDecStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int n_items = B * n_kv * ns;
  const int W = gridDim.x * kDecWarps;
  const int worker = blockIdx.x * kDecWarps + warp;

  // ---- load cursor: runs kDecStages chunks ahead over this warp's item stream
  DecItem li{};
  int l_item = worker, l_c = 0;
  auto skip_empty = [&]() {
    while (l_item < n_items) {
      li = dec_item(l_item, n_kv, ns, split, pos, max_len);
      if (li.nk > 0) return;
      l_item += W;
    }
  };
  auto issue = [&](int stage) {
    if (l_item >= n_items) return;
    if (lane == 0) {
      const int row = (int)kv_row(L, li.b, li.kvh, n_kv, max_len, li.k0 + l_c * kDecChunk);
      uint8_t* dst = ring + stage * kStageBytes;
      mbar_arrive_expect_tx(&full[stage], kStageBytes);
#pragma unroll
      for (int h = 0; h < H; ++h) {
        tma_load_2d(dst + h * kHalfBytes, &tmK, &full[stage], h * 64, row, kEvictFirst);
        tma_load_2d(dst + (H + h) * kHalfBytes, &tmV, &full[stage], h * 64, row, kEvictFirst);
      }
    }
    if (++l_c * kDecChunk >= li.nk) {
      l_c = 0;
      l_item += W;
      skip_empty();
    }
  };
  skip_empty();
#pragma unroll
  for (int s = 0; s < kDecStages; ++s) issue(s);

  const int g = lane >> 2;  // query-head row of this lane (rows >= G are padding)
  const int q2 = 2 * (lane & 3);
  int stage = 0;
  uint32_t phase = 0;
  for (int item = worker; item < n_items; item += W) {
    const DecItem it = dec_item(item, n_kv, ns, split, pos, max_len);
    const int sidx = item % ns;
    const int64_t obase = ((int64_t)it.b * n_q + it.kvh * G + g) * ns + sidx;
    if (it.nk == 0) {
      // an empty split (past the sequence): weight 0 in the merge, and its o row
      // zeroed so the merge never multiplies stale workspace bytes (possibly
      // NaN) by that zero weight
      if (g < G) {
        float* dst = ws_o + obase * D;
#pragma unroll
        for (int n = 0; n < NT; ++n) *reinterpret_cast<float2*>(dst + n * 8 + q2) = make_float2(0.f, 0.f);
        if ((lane & 3) == 0) {
          ws_ml[obase * 2] = -INFINITY;
          ws_ml[obase * 2 + 1] = 0.f;
        }
      }
      continue;
    }
    uint32_t qa[D / 16][2];
    {
      const __nv_bfloat16* qrow = qkv + (int64_t)it.b * ld + (int64_t)(it.kvh * G + g) * D;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + q2) : 0u;
        qa[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + q2) : 0u;
      }
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m = -INFINITY, l = 0.f;
    const int nch = (it.nk + kDecChunk - 1) / kDecChunk;
    for (int c = 0; c < nch; ++c) {
      mbar_wait(&full[stage], phase);
      const uint32_t kb = smem_u32(ring + stage * kStageBytes), vb = kb + H * kHalfBytes;
      // S = Q K^T over the chunk's 16 keys (two n8 tiles)
      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int mi = lane >> 3, key = (mi >> 1) * 8 + (lane & 7);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const int e = ks * 16 + (mi & 1) * 8;
          uint32_t b00, b01, b10, b11;
          ldsm_x4(kb + (e >> 6) * kHalfBytes + sw128(key, e & 63), b00, b01, b10, b11);
          mma_bf16_16816(s0, qa[ks][0], 0u, qa[ks][1], 0u, b00, b01);
          mma_bf16_16816(s1, qa[ks][0], 0u, qa[ks][1], 0u, b10, b11);
        }
      }
      // online softmax (base 2) on row g: keys c*16 + {q2, q2+1, 8+q2, 9+q2}
      const int kbase = c * kDecChunk + q2;
      float x0 = kbase < it.nk ? s0[0] * scale_log2 : -INFINITY;
      float x1 = kbase + 1 < it.nk ? s0[1] * scale_log2 : -INFINITY;
      float x2 = kbase + 8 < it.nk ? s1[0] * scale_log2 : -INFINITY;
      float x3 = kbase + 9 < it.nk ? s1[1] * scale_log2 : -INFINITY;
      float mx = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m, mx);
      const float alpha = exp2f(m - m_new);
      const float p0 = exp2f(x0 - m_new), p1 = exp2f(x1 - m_new), p2 = exp2f(x2 - m_new), p3 = exp2f(x3 - m_new);
      l = l * alpha + (p0 + p1) + (p2 + p3);
      m = m_new;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        o[n][0] *= alpha;
        o[n][1] *= alpha;
      }
      const uint32_t pa0 = pack_bf16x2(p0, p1), pa2 = pack_bf16x2(p2, p3);
      // O += P V (V rows = keys, ldmatrix.trans gives the k-major B fragments)
      {
        const int mi = lane >> 3, key = (mi & 1) * 8 + (lane & 7);
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          const int e = np * 16 + (mi >> 1) * 8;
          uint32_t v0, v1, v2, v3;
          ldsm_x4_t(vb + (e >> 6) * kHalfBytes + sw128(key, e & 63), v0, v1, v2, v3);
          mma_bf16_16816(o[2 * np], pa0, 0u, pa2, 0u, v0, v1);
          mma_bf16_16816(o[2 * np + 1], pa0, 0u, pa2, 0u, v2, v3);
        }
      }
      __syncwarp();
      issue(stage);  // refill the freed stage kDecStages chunks ahead
      if (++stage == kDecStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (g < G) {
      float* dst = ws_o + obase * D;
#pragma unroll
      for (int n = 0; n < NT; ++n) *reinterpret_cast<float2*>(dst + n * 8 + q2) = make_float2(o[n][0], o[n][1]);
      if ((lane & 3) == 0) {
        ws_ml[obase * 2] = m;
        ws_ml[obase * 2 + 1] = l;
      }
    }
  }
}

// Warp per (sequence, query head): lanes hold the split statistics (m, l),
// the max and the weighted denominator are warp reductions, and every lane
// accumulates D/32 output columns over the splits with all partial loads of a
// split in flight at once.  Splits with m = -inf (past the sequence) weigh 0.
// Many splits (small batches: few (sequence, kv head) items, so the key range
// is cut finely): one CTA of 8 warps per (sequence, q head); warp w folds splits
// w, w+8, ... and the 8 partial rows are summed in warp order (deterministic).
constexpr int kWideMergeWarps = 8;
__global__ void __launch_bounds__(kWideMergeWarps * 32) decode_merge_wide_kernel(
    const float* __restrict__ ws_o, const float* __restrict__ ws_ml, int n_splits, int n_q, int D,
    __nv_bfloat16* __restrict__ out, int64_t ldo) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[kWideMergeWarps];
  __shared__ float num_s[kWideMergeWarps][128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int item = blockIdx.x;
  const int b = item / n_q, hq = item - b * n_q;
  const int64_t base = (int64_t)item * n_splits;
  float M = -INFINITY;
  for (int s2 = tid; s2 < n_splits; s2 += blockDim.x) M = fmaxf(M, ws_ml[(base + s2) * 2]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) red[warp] = M;
  __syncthreads();
  M = red[0];
#pragma unroll
  for (int w = 1; w < kWideMergeWarps; ++w) M = fmaxf(M, red[w]);
  __syncthreads();
  float den = 0.f;
  for (int s2 = tid; s2 < n_splits; s2 += blockDim.x) {
    const float m = ws_ml[(base + s2) * 2];
    if (m != -INFINITY) den = fmaf(exp2f(m - M), ws_ml[(base + s2) * 2 + 1], den);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  if (lane == 0) red[warp] = den;
  __syncthreads();
  den = 0.f;
#pragma unroll
  for (int w = 0; w < kWideMergeWarps; ++w) den += red[w];
  const float inv = den > 0.f ? 1.f / den : 0.f;
  for (int db = 0; db < D; db += 128) {  // uniform trip count: the loop holds __syncthreads
    const int d0 = db + lane * 4;
    const bool act = d0 < D;
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int s2 = warp; act && s2 < n_splits; s2 += kWideMergeWarps) {
      const float m = ws_ml[(base + s2) * 2];
      if (m == -INFINITY) continue;
      const float wgt = exp2f(m - M);
      const float4 o4 = *reinterpret_cast<const float4*>(ws_o + (base + s2) * D + d0);
      num.x = fmaf(wgt, o4.x, num.x);
      num.y = fmaf(wgt, o4.y, num.y);
      num.z = fmaf(wgt, o4.z, num.z);
      num.w = fmaf(wgt, o4.w, num.w);
    }
    __syncthreads();
    *reinterpret_cast<float4*>(&num_s[warp][lane * 4]) = num;
    __syncthreads();
    if (warp == 0 && act) {
      float4 t = *reinterpret_cast<const float4*>(&num_s[0][lane * 4]);
#pragma unroll
      for (int w = 1; w < kWideMergeWarps; ++w) {
        const float4 u = *reinterpret_cast<const float4*>(&num_s[w][lane * 4]);
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
      __nv_bfloat16* orow = out + (int64_t)b * ldo + (int64_t)hq * D + d0;
      *reinterpret_cast<uint2*>(orow) =
          make_uint2(pack_bf16x2(t.x * inv, t.y * inv), pack_bf16x2(t.z * inv, t.w * inv));
    }
  }
}

constexpr int kMergeWarps = 4;
__global__ void __launch_bounds__(kMergeWarps * 32) decode_merge_kernel(const float* __restrict__ ws_o,
                                                                        const float* __restrict__ ws_ml, int n_splits,
                                                                        int n_q, int B, int D,
                                                                        __nv_bfloat16* __restrict__ out, int64_t ldo) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
  if (item >= B * n_q) return;
  const int b = item / n_q, hq = item - b * n_q;
  const int64_t base = (int64_t)item * n_splits;  // == (b * n_q + hq) * n_splits
  if (n_splits <= 32 && D == 128) {
    // one split per lane: the (m, l) pairs and the first 8 partial rows are
    // all requested before any reduction, so the merge costs ~2 memory round
    // trips instead of one per dependent pass
    constexpr int kPre = 8;
    const int d0 = lane * 4;
    float4 pre[kPre];
#pragma unroll
    for (int s2 = 0; s2 < kPre; ++s2)
      pre[s2] = s2 < n_splits ? *reinterpret_cast<const float4*>(ws_o + (base + s2) * D + d0)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
    const float m = lane < n_splits ? ws_ml[(base + lane) * 2] : -INFINITY;
    const float l = lane < n_splits ? ws_ml[(base + lane) * 2 + 1] : 0.f;
    float M = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float wgt = m != -INFINITY ? exp2f(m - M) : 0.f;
    float den = wgt * l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    const float inv = den > 0.f ? 1.f / den : 0.f;
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s2 = 0; s2 < kPre; ++s2) {
      const float w2 = __shfl_sync(0xffffffffu, wgt, s2);
      if (s2 < n_splits) {
        num.x = fmaf(w2, pre[s2].x, num.x);
        num.y = fmaf(w2, pre[s2].y, num.y);
        num.z = fmaf(w2, pre[s2].z, num.z);
        num.w = fmaf(w2, pre[s2].w, num.w);
      }
    }
#pragma unroll 4
    for (int s2 = kPre; s2 < n_splits; ++s2) {
      const float w2 = __shfl_sync(0xffffffffu, wgt, s2);
      const float4 o4 = *reinterpret_cast<const float4*>(ws_o + (base + s2) * D + d0);
      num.x = fmaf(w2, o4.x, num.x);
      num.y = fmaf(w2, o4.y, num.y);
      num.z = fmaf(w2, o4.z, num.z);
      num.w = fmaf(w2, o4.w, num.w);
    }
    __nv_bfloat16* orow = out + (int64_t)b * ldo + (int64_t)hq * D + d0;
    *reinterpret_cast<uint2*>(orow) =
        make_uint2(pack_bf16x2(num.x * inv, num.y * inv), pack_bf16x2(num.z * inv, num.w * inv));
    return;
  }
  float M = -INFINITY;
  for (int s2 = lane; s2 < n_splits; s2 += 32) M = fmaxf(M, ws_ml[(base + s2) * 2]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float den = 0.f;
  for (int s2 = lane; s2 < n_splits; s2 += 32) {
    const float m = ws_ml[(base + s2) * 2];
    if (m != -INFINITY) den = fmaf(exp2f(m - M), ws_ml[(base + s2) * 2 + 1], den);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  const float inv = den > 0.f ? 1.f / den : 0.f;
  for (int d0 = lane * 4; d0 < D; d0 += 128) {
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int s2 = 0; s2 < n_splits; ++s2) {
      const float m = ws_ml[(base + s2) * 2];  // same address in every lane
      if (m == -INFINITY) continue;
      const float wgt = exp2f(m - M);
      const float4 o4 = *reinterpret_cast<const float4*>(ws_o + (base + s2) * D + d0);
      num.x = fmaf(wgt, o4.x, num.x);
      num.y = fmaf(wgt, o4.y, num.y);
      num.z = fmaf(wgt, o4.z, num.z);
      num.w = fmaf(wgt, o4.w, num.w);
    }
    __nv_bfloat16* orow = out + (int64_t)b * ldo + (int64_t)hq * D + d0;
    *reinterpret_cast<uint2*>(orow) = make_uint2(pack_bf16x2(num.x * inv, num.y * inv), pack_bf16x2(num.z * inv, num.w * inv));
  }
}

}  // namespace attn
}  // namespace hap

namespace hap {
namespace attn {
// Prefill: copy every token's (post-RoPE) k and v from the fused qkv rows into
// the head-major cache rows [0, seq_len) of its sequence.
template <int D>
__global__ void kv_fill_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, int n_q, int n_kv, int S,
                               __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int max_len,
                               KvLayout L) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x, b = blockIdx.y;
  if (kv_row(L, b, 0, n_kv, max_len, i) < 0) return;  // page not allocated
  const __nv_bfloat16* row = qkv + ((int64_t)b * S + i) * ld;
  for (int v = threadIdx.x; v < n_kv * D / 8; v += blockDim.x) {
    const int hh = v / (D / 8), c = (v % (D / 8)) * 8;
    const int64_t dst = kv_row(L, b, hh, n_kv, max_len, i) * D + c;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + hh) * D + c);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + n_kv + hh) * D + c);
  }
}
}  // namespace attn
}  // namespace hap

using namespace hap;
using namespace hap::attn;

static int kv_cache_fill(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                         int64_t n_kv_heads, int64_t head_dim, void* k_cache, void* v_cache, int64_t max_len,
                         KvLayout L, void* stream) {
  if (!qkv || !k_cache || !v_cache || n_seqs < 0 || seq_len < 0 || n_q_heads < 1 || n_kv_heads < 1)
    return HAP_ERR_INVALID_ARG;
  if (seq_len > max_len) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  if (ldqkv % 8 || ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(k_cache) |
                     reinterpret_cast<uintptr_t>(v_cache)) & 15))
    return HAP_ERR_MISALIGNED;
  if (n_seqs == 0 || seq_len == 0) return HAP_OK;
  dim3 grid((unsigned)seq_len, (unsigned)n_seqs);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto* q = reinterpret_cast<const __nv_bfloat16*>(qkv);
  auto* kc = reinterpret_cast<__nv_bfloat16*>(k_cache);
  auto* vc = reinterpret_cast<__nv_bfloat16*>(v_cache);
  if (head_dim == 128)
    { if (hap::launch_k(kv_fill_kernel<128>, dim3(grid), dim3(128), 0, st, q, ldqkv, (int)n_q_heads, (int)n_kv_heads, (int)seq_len, kc, vc, (int)max_len, L) != cudaSuccess) return HAP_ERR_LAUNCH; }
  else
    { if (hap::launch_k(kv_fill_kernel<64>, dim3(grid), dim3(128), 0, st, q, ldqkv, (int)n_q_heads, (int)n_kv_heads, (int)seq_len, kc, vc, (int)max_len, L) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_kv_cache_fill(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                                 int64_t n_kv_heads, int64_t head_dim, void* k_cache, void* v_cache, int64_t max_len,
                                 void* stream) {
  return kv_cache_fill(qkv, ldqkv, n_seqs, seq_len, n_q_heads, n_kv_heads, head_dim, k_cache, v_cache, max_len,
                       KvLayout{nullptr, 0, 0}, stream);
}

static bool paged_ok(const int32_t* block_table, int64_t max_pages, int64_t page_size) {
  return block_table && max_pages >= 1 && page_size >= kDecChunk && page_size % kDecChunk == 0;
}

extern "C" int hap_kv_cache_fill_paged(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len,
                                       int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim, void* k_pool,
                                       void* v_pool, const int32_t* block_table, int64_t max_pages,
                                       int64_t page_size, void* stream) {
  if (!paged_ok(block_table, max_pages, page_size)) return HAP_ERR_INVALID_ARG;
  return kv_cache_fill(qkv, ldqkv, n_seqs, seq_len, n_q_heads, n_kv_heads, head_dim, k_pool, v_pool,
                       max_pages * page_size, KvLayout{block_table, (int)max_pages, (int)page_size}, stream);
}

extern "C" size_t hap_attn_prefill_workspace_bytes(void) { return hap::attn_prefill_tc_workspace_bytes(); }

extern "C" int hap_attn_prefill(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                void* out, int64_t ldo, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                                int64_t n_kv_heads, int64_t head_dim, float scale, int32_t causal, void* workspace,
                                size_t ws_bytes, void* stream) {
  if (!q || !k || !v || !out || n_seqs < 0 || seq_len < 0 || n_q_heads < 1 || n_kv_heads < 1) return HAP_ERR_INVALID_ARG;
  if (!workspace || ws_bytes < hap::attn_prefill_tc_workspace_bytes()) return HAP_ERR_WORKSPACE;
  if (reinterpret_cast<uintptr_t>(workspace) & 3) return HAP_ERR_MISALIGNED;
  if (n_q_heads % n_kv_heads) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  if (ldq % 8 || ldk % 8 || ldv % 8 || ldo % 8) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15)
    return HAP_ERR_MISALIGNED;
  if (n_seqs == 0 || seq_len == 0) return HAP_OK;
  return hap::attn_prefill_tc(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, seq_len, n_q_heads, n_kv_heads, head_dim,
                              scale, causal, reinterpret_cast<int*>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

// Key-split size for the warp-pipelined decode: items = B * n_kv * ceil(len/split)
// spread round-robin over 148 x kDecWarps warp workers; minimise
// rounds x (chunks per item + ~1 chunk of per-item overhead), with at most 32
// splits per (sequence, head) so the merge is the one-split-per-lane kernel
// (small batches otherwise cut the keys into 16-key splits whose merge reads
// more partials than the cache holds: Qwen2-57B B=1, 128 splits, merge 12 us).
static void plan_decode(int64_t B, int64_t n_kv, int64_t max_len, int* split, int* ns) {
  const int64_t workers = (int64_t)kNumSMs * kDecWarps;
  const int64_t cps = (max_len + kDecChunk - 1) / kDecChunk;
  int64_t best_sc = cps, best_cost = INT64_MAX;
  for (int64_t sc = 1; sc <= cps; ++sc) {
    const int64_t n = (cps + sc - 1) / sc;
    if (sc > 1 && (cps + sc - 2) / (sc - 1) == n) continue;  // same split count as a smaller sc
    if (n > 32) continue;
    const int64_t rounds = (B * n_kv * n + workers - 1) / workers;
    const int64_t cost = rounds * (sc + 1);
    if (cost < best_cost) {
      best_cost = cost;
      best_sc = sc;
    }
  }
  *split = (int)(best_sc * kDecChunk);
  *ns = (int)((max_len + best_sc * kDecChunk - 1) / (best_sc * kDecChunk));
}

extern "C" size_t hap_attn_decode_workspace_bytes(int64_t B, int64_t n_q_heads, int64_t head_dim, int64_t max_len) {
  if (B < 0 || n_q_heads < 1 || head_dim < 1 || max_len < 1) return 0;
  // the split count depends on n_kv (unknown here): take the largest over every
  // kv-head count that divides n_q
  int64_t n = 1;
  for (int64_t nkv = 1; nkv <= n_q_heads; ++nkv) {
    if (n_q_heads % nkv) continue;
    int split, ns;
    plan_decode(B, nkv, max_len, &split, &ns);
    if (ns > n) n = ns;
  }
  return (size_t)(B * n_q_heads * n) * (size_t)(head_dim + 2) * sizeof(float);
}

template <int D>
static int launch_decode(const __nv_bfloat16* q, int64_t ldqkv, __nv_bfloat16* kc, __nv_bfloat16* vc, int64_t max_len,
                         const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads, float scale,
                         float* ws_o, float* ws_ml, int* ns_out, KvLayout L, uint64_t cache_rows, cudaStream_t st) {
  const int G = (int)(n_q_heads / n_kv_heads);
  { if (hap::launch_kr(B, kv_append_kernel<D>, dim3((unsigned)B), dim3(128), 0, st, q, ldqkv, (int)n_q_heads, (int)n_kv_heads, kc, vc, (int)max_len, pos, L) != cudaSuccess) return HAP_ERR_LAUNCH; }
  const float sl2 = scale * 1.4426950408889634f;
  int split, ns;
  plan_decode(B, n_kv_heads, max_len, &split, &ns);
  *ns_out = ns;  // <= the count hap_attn_decode_workspace_bytes provisions for
  const uint64_t rows = cache_rows;
  CUtensorMap tmK, tmV;
  if (!encode_tmap_2d_bf16(&tmK, kc, D, rows, D * 2, 64, kDecChunk, true) ||
      !encode_tmap_2d_bf16(&tmV, vc, D, rows, D * 2, 64, kDecChunk, true))
    return HAP_ERR_DRIVER;
  const int smem = kDecWarps * kDecStages * 2 * (D / 64) * kDecChunk * 128 + 1024;
  const int64_t items = B * n_kv_heads * ns;
  const int64_t ctas = (items + kDecWarps - 1) / kDecWarps;
  const unsigned grid = (unsigned)(ctas < kNumSMs ? ctas : kNumSMs);
#define HAP_DEC_CASE(GG)                                                                                          \
  case GG: {                                                                                                      \
    static bool cfg = false;                                                                                      \
    if (!cfg) {                                                                                                   \
      if (configure_smem((const void*)decode_mma_kernel<D, GG>, smem) != 0) return HAP_ERR_LAUNCH;                \
      cfg = true;                                                                                                 \
    }                                                                                                             \
    { if (hap::launch_kr(B, decode_mma_kernel<D, GG>, dim3(grid), dim3(kDecWarps * 32), smem, st, tmK, tmV, q, ldqkv, (int)max_len, pos, (int)B,   \
                                                                 (int)n_q_heads, (int)n_kv_heads, sl2, ws_o,      \
                                                                 ws_ml, ns, split, L) != cudaSuccess) return HAP_ERR_LAUNCH; }                            \
    break;                                                                                                        \
  }
  switch (G) {
    HAP_DEC_CASE(1)
    HAP_DEC_CASE(2)
    HAP_DEC_CASE(3)
    HAP_DEC_CASE(4)
    HAP_DEC_CASE(5)
    HAP_DEC_CASE(6)
    HAP_DEC_CASE(7)
    HAP_DEC_CASE(8)
    default: return HAP_ERR_UNSUPPORTED;
  }
#undef HAP_DEC_CASE
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

static int attn_decode(const void* qkv, int64_t ldqkv, void* k_cache, void* v_cache, int64_t max_len,
                       const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim,
                       float scale, void* out, int64_t ldo, void* workspace, size_t ws_bytes, KvLayout L,
                       uint64_t cache_rows, void* stream) {
  if (!qkv || !k_cache || !v_cache || !pos || !out || B < 0 || max_len < 1 || n_q_heads < 1 || n_kv_heads < 1)
    return HAP_ERR_INVALID_ARG;
  if (n_q_heads % n_kv_heads) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  const int G = (int)(n_q_heads / n_kv_heads);
  if (G > kMaxG) return HAP_ERR_UNSUPPORTED;
  if (ldqkv % 8 || ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(k_cache) |
                     reinterpret_cast<uintptr_t>(v_cache)) & 15))
    return HAP_ERR_MISALIGNED;
  if (B == 0) return HAP_OK;
  const size_t need = hap_attn_decode_workspace_bytes(B, n_q_heads, head_dim, max_len);
  if (!workspace || ws_bytes < need) return HAP_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // ws_ml sits after the largest o block the workspace size accounts for
  const size_t n_units = need / ((size_t)(head_dim + 2) * sizeof(float));
  float* ws_o = reinterpret_cast<float*>(workspace);
  float* ws_ml = ws_o + n_units * head_dim;
  int ns = 0;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(qkv);
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(k_cache);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(v_cache);
  const int rc = head_dim == 128 ? launch_decode<128>(q, ldqkv, kc, vc, max_len, pos, B, n_q_heads, n_kv_heads, scale, ws_o, ws_ml, &ns, L, cache_rows, st)
                                 : launch_decode<64>(q, ldqkv, kc, vc, max_len, pos, B, n_q_heads, n_kv_heads, scale, ws_o, ws_ml, &ns, L, cache_rows, st);
  if (rc != HAP_OK) return rc;
  if (ns > 32) {
    if (hap::launch_kr(B, decode_merge_wide_kernel, dim3((unsigned)(B * n_q_heads)), dim3(kWideMergeWarps * 32), 0, st,
                      ws_o, ws_ml, ns, (int)n_q_heads, (int)head_dim, reinterpret_cast<__nv_bfloat16*>(out),
                      ldo) != cudaSuccess)
      return HAP_ERR_LAUNCH;
  } else {
    if (hap::launch_kr(B, decode_merge_kernel, dim3((unsigned)((B * n_q_heads + kMergeWarps - 1) / kMergeWarps)),
                      dim3(kMergeWarps * 32), 0, st, ws_o, ws_ml, ns, (int)n_q_heads, (int)B, (int)head_dim,
                      reinterpret_cast<__nv_bfloat16*>(out), ldo) != cudaSuccess)
      return HAP_ERR_LAUNCH;
  }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_attn_decode(const void* qkv, int64_t ldqkv, void* k_cache, void* v_cache, int64_t max_len,
                               const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads,
                               int64_t head_dim, float scale, void* out, int64_t ldo, void* workspace,
                               size_t ws_bytes, void* stream) {
  return attn_decode(qkv, ldqkv, k_cache, v_cache, max_len, pos, B, n_q_heads, n_kv_heads, head_dim, scale, out, ldo,
                     workspace, ws_bytes, KvLayout{nullptr, 0, 0}, (uint64_t)(B * n_kv_heads * max_len), stream);
}

extern "C" int hap_attn_decode_paged(const void* qkv, int64_t ldqkv, void* k_pool, void* v_pool, int64_t n_pages,
                                     int64_t page_size, const int32_t* block_table, int64_t max_pages,
                                     const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads,
                                     int64_t head_dim, float scale, void* out, int64_t ldo, void* workspace,
                                     size_t ws_bytes, void* stream) {
  if (!paged_ok(block_table, max_pages, page_size) || n_pages < 1) return HAP_ERR_INVALID_ARG;
  return attn_decode(qkv, ldqkv, k_pool, v_pool, max_pages * page_size, pos, B, n_q_heads, n_kv_heads, head_dim,
                     scale, out, ldo, workspace, ws_bytes, KvLayout{block_table, (int)max_pages, (int)page_size},
                     (uint64_t)(n_pages * n_kv_heads * page_size), stream);
}
