// Attention core entry points: causal GQA prefill (tcgen05 flash attention,
// attn_tc.cu) and split-KV GQA decode over a head-major KV cache.
//
// Decode: one CTA per (kv-head, 256-key split, sequence) streams K and V once
// (16-byte coalesced rows, several loads in flight per thread) for all
// G = n_q/n_kv query heads of the group, writes fp32 partial (o, m, l), and a
// merge kernel rescales the splits.  KV cache layout: [B, n_kv, max_len, d].
//
// Models: score+value term 4*n*kv_len*h of attention_flops (reference
// arch.py:161); decode kv_len = input_len + output_len//2 (planner.py:226).
#include "common.cuh"

namespace hap {
int attn_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                    int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, int64_t head_dim, float scale,
                    int32_t causal, cudaStream_t st);

namespace attn {

constexpr int kThreads = 128;

// ------------------------------------------------------------------ decode --
constexpr int kSplit = 256;
constexpr int kMaxG = 8;

// Copy the new token's k and v (from the fused qkv row, after RoPE) into the cache.
template <int D>
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, int n_q, int n_kv,
                                 __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int max_len,
                                 const int32_t* __restrict__ pos) {
  const int b = blockIdx.x;
  const int p = pos[b];
  const __nv_bfloat16* row = qkv + (int64_t)b * ld;
  for (int i = threadIdx.x; i < n_kv * D / 8; i += blockDim.x) {
    const int hh = i / (D / 8), c = (i % (D / 8)) * 8;
    const int64_t dst = (((int64_t)b * n_kv + hh) * max_len + p) * D + c;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + hh) * D + c);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + n_kv + hh) * D + c);
  }
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads) decode_split_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld,
                                                                const __nv_bfloat16* __restrict__ kc,
                                                                const __nv_bfloat16* __restrict__ vc, int max_len,
                                                                const int32_t* __restrict__ pos, int n_q, int n_kv,
                                                                float scale_log2, float* __restrict__ ws_o,
                                                                float* __restrict__ ws_ml, int n_splits) {
  constexpr int LPK = D / 8;              // lanes per key row (16 B each)
  constexpr int KPP = kThreads / LPK;     // keys per CTA pass
  constexpr int U = 4;                    // passes in flight per thread
  __shared__ float qs[G][D];
  __shared__ float sc[G][kSplit];
  __shared__ float red[KPP][G][D];
  __shared__ float mstat[G], lstat[G];
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int L = pos[b] + 1;
  const int k0 = split * kSplit;
  const int k1 = min(L, k0 + kSplit);
  const int nk = k1 - k0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t out_base = (((int64_t)b * n_q + (int64_t)kvh * G) * n_splits + split);
  if (nk <= 0) {
    if (threadIdx.x < G) {
      float* ml = ws_ml + (out_base + (int64_t)threadIdx.x * n_splits) * 2;
      ml[0] = -INFINITY;
      ml[1] = 0.f;
    }
    return;
  }
  for (int i = threadIdx.x; i < G * D; i += kThreads) {
    const int gg = i / D, d = i % D;
    qs[gg][d] = __bfloat162float(qkv[(int64_t)b * ld + (int64_t)(kvh * G + gg) * D + d]);
  }
  __syncthreads();
  const __nv_bfloat16* kbase = kc + (((int64_t)b * n_kv + kvh) * max_len + k0) * D;
  const __nv_bfloat16* vbase = vc + (((int64_t)b * n_kv + kvh) * max_len + k0) * D;
  const int kr = threadIdx.x / LPK;   // key slot within a pass
  const int l16 = threadIdx.x % LPK;  // 8-dim slice
  float qreg[G][8];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int i = 0; i < 8; ++i) qreg[gg][i] = qs[gg][l16 * 8 + i];

  // ---- scores: U passes of KPP keys in flight
  for (int kb = 0; kb < nk; kb += KPP * U) {
    uint4 kv4[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * KPP + kr;
      kv4[u] = kk < nk ? __ldg(reinterpret_cast<const uint4*>(kbase + (int64_t)kk * D + l16 * 8))
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * KPP + kr;
      const uint32_t kw[4] = {kv4[u].x, kv4[u].y, kv4[u].z, kv4[u].w};
      float kf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(kw[i]);
        kf[2 * i] = f.x;
        kf[2 * i + 1] = f.y;
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(qreg[gg][i], kf[i], acc);
#pragma unroll
        for (int o2 = LPK / 2; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
        if (l16 == 0 && kk < nk) sc[gg][kk] = acc * scale_log2;
      }
    }
  }
  __syncthreads();
  // ---- softmax statistics per query head
  for (int gg = warp; gg < G; gg += kThreads / 32) {
    float m = -INFINITY;
    for (int i = lane; i < nk; i += 32) m = fmaxf(m, sc[gg][i]);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o2));
    float l = 0.f;
    for (int i = lane; i < nk; i += 32) {
      const float p = exp2f(sc[gg][i] - m);
      sc[gg][i] = p;
      l += p;
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
    if (lane == 0) {
      mstat[gg] = m;
      lstat[gg] = l;
    }
  }
  __syncthreads();
  // ---- O = P V: thread owns an 8-dim slice of key slot kr, U rows in flight
  float acc[G][8];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[gg][i] = 0.f;
  for (int kb = 0; kb < nk; kb += KPP * U) {
    uint4 vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * KPP + kr;
      vv[u] = kk < nk ? __ldg(reinterpret_cast<const uint4*>(vbase + (int64_t)kk * D + l16 * 8))
                      : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * KPP + kr;
      if (kk >= nk) continue;
      const uint32_t vw[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
      float vf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(vw[i]);
        vf[2 * i] = f.x;
        vf[2 * i + 1] = f.y;
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const float p = sc[gg][kk];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[gg][i] = fmaf(p, vf[i], acc[gg][i]);
      }
    }
  }
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int i = 0; i < 8; ++i) red[kr][gg][l16 * 8 + i] = acc[gg][i];
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += kThreads) {
    const int gg = i / D, d = i % D;
    float sacc = 0.f;
#pragma unroll
    for (int q2 = 0; q2 < KPP; ++q2) sacc += red[q2][gg][d];
    ws_o[(out_base + (int64_t)gg * n_splits) * D + d] = sacc;
  }
  if (threadIdx.x < G) {
    float* ml = ws_ml + (out_base + (int64_t)threadIdx.x * n_splits) * 2;
    ml[0] = mstat[threadIdx.x];
    ml[1] = lstat[threadIdx.x];
  }
}

__global__ void decode_merge_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_ml, int n_splits,
                                    int n_q, int D, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int hq = blockIdx.x, b = blockIdx.y;
  const int64_t base = ((int64_t)b * n_q + hq) * n_splits;
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, ws_ml[(base + s) * 2]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float num = 0.f, den = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float m = ws_ml[(base + s) * 2];
      if (m == -INFINITY) continue;
      const float w = exp2f(m - M);
      num = fmaf(w, ws_o[(base + s) * D + d], num);
      den = fmaf(w, ws_ml[(base + s) * 2 + 1], den);
    }
    out[(int64_t)b * ldo + (int64_t)hq * D + d] = __float2bfloat16_rn(den > 0.f ? num / den : 0.f);
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
                               __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int max_len) {
  const int i = blockIdx.x, b = blockIdx.y;
  const __nv_bfloat16* row = qkv + ((int64_t)b * S + i) * ld;
  for (int v = threadIdx.x; v < n_kv * D / 8; v += blockDim.x) {
    const int hh = v / (D / 8), c = (v % (D / 8)) * 8;
    const int64_t dst = (((int64_t)b * n_kv + hh) * max_len + i) * D + c;
    *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + hh) * D + c);
    *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(row + (int64_t)(n_q + n_kv + hh) * D + c);
  }
}
}  // namespace attn
}  // namespace hap

using namespace hap::attn;

extern "C" int hap_kv_cache_fill(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                                 int64_t n_kv_heads, int64_t head_dim, void* k_cache, void* v_cache, int64_t max_len,
                                 void* stream) {
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
    kv_fill_kernel<128><<<grid, 128, 0, st>>>(q, ldqkv, (int)n_q_heads, (int)n_kv_heads, (int)seq_len, kc, vc, (int)max_len);
  else
    kv_fill_kernel<64><<<grid, 128, 0, st>>>(q, ldqkv, (int)n_q_heads, (int)n_kv_heads, (int)seq_len, kc, vc, (int)max_len);
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_attn_prefill(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                void* out, int64_t ldo, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                                int64_t n_kv_heads, int64_t head_dim, float scale, int32_t causal, void* stream) {
  if (!q || !k || !v || !out || n_seqs < 0 || seq_len < 0 || n_q_heads < 1 || n_kv_heads < 1) return HAP_ERR_INVALID_ARG;
  if (n_q_heads % n_kv_heads) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  if (ldq % 8 || ldk % 8 || ldv % 8 || ldo % 8) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15)
    return HAP_ERR_MISALIGNED;
  if (n_seqs == 0 || seq_len == 0) return HAP_OK;
  return hap::attn_prefill_tc(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, seq_len, n_q_heads, n_kv_heads, head_dim,
                              scale, causal, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" size_t hap_attn_decode_workspace_bytes(int64_t B, int64_t n_q_heads, int64_t head_dim, int64_t max_len) {
  if (B < 0 || n_q_heads < 1 || head_dim < 1 || max_len < 1) return 0;
  const int64_t ns = (max_len + kSplit - 1) / kSplit;
  return (size_t)(B * n_q_heads * ns) * (size_t)(head_dim + 2) * sizeof(float);
}

template <int D>
static int launch_decode(const __nv_bfloat16* q, int64_t ldqkv, __nv_bfloat16* kc, __nv_bfloat16* vc, int64_t max_len,
                         const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads, float scale,
                         float* ws_o, float* ws_ml, int ns, cudaStream_t st) {
  const int G = (int)(n_q_heads / n_kv_heads);
  kv_append_kernel<D><<<(unsigned)B, 128, 0, st>>>(q, ldqkv, (int)n_q_heads, (int)n_kv_heads, kc, vc, (int)max_len, pos);
  dim3 grid((unsigned)ns, (unsigned)n_kv_heads, (unsigned)B);
  const float sl2 = scale * 1.4426950408889634f;
#define HAP_DEC_CASE(GG)                                                                                          \
  case GG:                                                                                                        \
    decode_split_kernel<D, GG><<<grid, kThreads, 0, st>>>(q, ldqkv, kc, vc, (int)max_len, pos, (int)n_q_heads,    \
                                                          (int)n_kv_heads, sl2, ws_o, ws_ml, ns);                 \
    break;
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

extern "C" int hap_attn_decode(const void* qkv, int64_t ldqkv, void* k_cache, void* v_cache, int64_t max_len,
                               const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads,
                               int64_t head_dim, float scale, void* out, int64_t ldo, void* workspace,
                               size_t ws_bytes, void* stream) {
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
  const int ns = (int)((max_len + kSplit - 1) / kSplit);
  float* ws_o = reinterpret_cast<float*>(workspace);
  float* ws_ml = ws_o + (size_t)B * n_q_heads * ns * head_dim;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(qkv);
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(k_cache);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(v_cache);
  const int rc = head_dim == 128 ? launch_decode<128>(q, ldqkv, kc, vc, max_len, pos, B, n_q_heads, n_kv_heads, scale, ws_o, ws_ml, ns, st)
                                 : launch_decode<64>(q, ldqkv, kc, vc, max_len, pos, B, n_q_heads, n_kv_heads, scale, ws_o, ws_ml, ns, st);
  if (rc != HAP_OK) return rc;
  decode_merge_kernel<<<dim3((unsigned)n_q_heads, (unsigned)B), 128, 0, st>>>(ws_o, ws_ml, ns, (int)n_q_heads, (int)head_dim,
                                                                              reinterpret_cast<__nv_bfloat16*>(out), ldo);
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
