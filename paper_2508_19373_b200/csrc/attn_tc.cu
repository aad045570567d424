// Causal GQA prefill attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA per (128-query tile, q head, sequence); 8 warps:
//   warp 0      TMA producer: Q once, then K_j / V_j 128-key tiles into a
//               2-stage ring (128B-swizzled, K-major Q/K, MN-major V)
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into a double-buffered
//               TMEM S tile (128x128 fp32), then O += P_{j-1} V_{j-1} into the
//               TMEM O accumulator (128 x d fp32), so S_{j+1} overlaps the
//               softmax of tile j and PV_j overlaps the softmax of tile j+1
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7  softmax + epilogue: thread = one query row (its TMEM lane);
//               tcgen05.ld the S row, causal mask, exp2-domain online softmax
//               with a lazily updated running max (O is rescaled in TMEM only
//               when the max grows by > 2^8 — exact, as the same stale max is
//               used for P and l), P written as bf16 into a swizzled K-major
//               smem tile that is the A operand of the PV MMA
// Final: O row / l -> bf16 -> global.
//
// Models: score+value term 4*n*kv_len*h of attention_flops (reference
// arch.py:161); causal: tiles above the diagonal are skipped.
#include "common.cuh"

namespace hap {
namespace attn_tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int kThreads = 384;  // 4 role warps + 2 softmax warpgroups
constexpr int kChunkBytes = 128 * 128;  // 128 rows x 128 B (64 bf16) swizzle-atom column
constexpr float kRescaleThreshold = 8.0f;  // log2 domain

template <int D>
struct Smem {
  static constexpr int kQ = (D / 64) * kChunkBytes;
  static constexpr int kK = (D / 64) * kChunkBytes;
  static constexpr int kV = (D / 64) * kChunkBytes;
  static constexpr int kP = (BN / 64) * kChunkBytes;
  static constexpr int kTotal = kQ + 2 * kK + 2 * kV + 1024;  // P lives in TMEM
};

// MN-major operand, 128B swizzle: MN chunks of 64 elements lbo bytes apart,
// 8-row K groups 1024 B apart.
__device__ __forceinline__ uint64_t make_sdesc_mn_sw128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 2^x on the FMA pipe (B200's SFU issues only ~8 ex2/clk/SM, the softmax's
// bottleneck): round-to-nearest split x = n + f via the 1.5*2^23 trick, a
// degree-3 minimax polynomial for 2^f on [-0.5, 0.5] (max rel err 1.4e-4,
// far below the bf16 rounding of P), and n added to the exponent bits.
// x is clamped at -125 so masked (-inf) scores give ~2e-38 instead of 0.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.05502926558256149f, 0.2422569841146469f);
  p = fmaf(f, p, 0.6932530403137207f);
  p = fmaf(f, p, 0.9999513626098633f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// D[tmem] (+)= A[tmem] * B[smem]^T (A = P, bf16 pairs packed per 32-bit column).
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t desc_b, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int64_t ldo, int S,
                   int n_q, int n_kv, float scale_log2, int causal) {
  pdl_trigger();
  pdl_wait();
  using SM = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + SM::kQ;           // [2][kK]
  uint8_t* sV = sK + 2 * SM::kK;       // [2][kV]

  __shared__ __align__(8) uint64_t q_full;
  __shared__ __align__(8) uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  __shared__ __align__(8) uint64_t s_full[2], s_free[2];
  __shared__ __align__(8) uint64_t p_full[2], o_done[2];
  __shared__ __align__(8) uint64_t o_final;
  __shared__ uint32_t tmem_base_s;
  __shared__ float red_max[2][2][BM];  // [tile parity][warpgroup][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_mblk = (S + BM - 1) / BM;
  const int mb = causal ? (n_mblk - 1 - (int)blockIdx.x) : (int)blockIdx.x;
  const int head = blockIdx.y, seq = blockIdx.z;
  const int kvh = head / (n_q / n_kv);
  const int q0 = mb * BM;
  const int tok0 = seq * S;
  const int kv_end = causal ? min(S, q0 + BM) : S;
  const int nt = (kv_end + BN - 1) / BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(&q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 256);
      mbar_init(&p_full[i], 256);
      mbar_init(&o_done[i], 1);
    }
    mbar_init(&o_final, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&tmem_base_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    // ===================== TMA producer: Q, then the K ring =====================
    // K_j is consumed by S_j only, so its stage is released as soon as S_j
    // completes and K runs ahead of V (separate ring, separate thread).
    if (lane == 0) {
      mbar_arrive_expect_tx(&q_full, SM::kQ);
      for (int c = 0; c < D / 64; ++c)
        tma_load_2d(sQ + c * kChunkBytes, &tmQ, &q_full, head * D + c * 64, tok0 + q0, kEvictFirst);
      for (int j = 0; j < nt; ++j) {
        const int s = j & 1;
        mbar_wait(&k_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], SM::kK);
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(sK + s * SM::kK + c * kChunkBytes, &tmK, &k_full[s], kvh * D + c * 64, tok0 + j * BN,
                      kEvictLast);
      }
    }
  } else if (warp == 3) {
    // ===================== TMA producer: the V ring (released after PV_j) =====================
    if (lane == 0) {
      for (int j = 0; j < nt; ++j) {
        const int s = j & 1;
        mbar_wait(&v_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[s], SM::kV);
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(sV + s * SM::kV + c * kChunkBytes, &tmV, &v_full[s], kvh * D + c * 64, tok0 + j * BN,
                      kEvictLast);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idS = make_idesc_bf16(BM, BN);
      const uint32_t idPV = make_idesc_bf16(BM, D) | (1u << 16);  // B (V) is MN-major
      mbar_wait(&q_full, 0);
      auto issue_pv = [&](int jp) {
        const int bp = jp & 1;
        mbar_wait(&v_full[jp & 1], (jp >> 1) & 1);
        mbar_wait(&p_full[bp], (jp >> 1) & 1);
        tc_fence_after();
        const uint32_t vbase = smem_u32(sV + (jp & 1) * SM::kV);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // P_jp sits in its S buffer: warpgroup w's 64 keys packed into columns [w*64, w*64+32)
          const uint32_t ta = tS[bp] + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint64_t db = make_sdesc_mn_sw128(vbase + kk * 16 * 128, kChunkBytes);
          umma_bf16_ts(tO, ta, db, idPV, (jp | kk) != 0);
        }
        umma_commit(&o_done[bp]);
        umma_commit(&v_empty[jp & 1]);
      };
      for (int j = 0; j < nt; ++j) {
        const int s = j & 1;
        mbar_wait(&k_full[s], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t qbase = smem_u32(sQ);
        const uint32_t kbase = smem_u32(sK + s * SM::kK);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = make_sdesc_sw128(qbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
          const uint64_t db = make_sdesc_sw128(kbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
          umma_bf16_ss(tS[s], da, db, idS, kk != 0);
        }
        umma_commit(&s_full[s]);
        umma_commit(&k_empty[s]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nt - 1);
      umma_commit(&o_final);
    }
  } else if (warp >= 4) {
    // ===================== softmax + epilogue =====================
    // Two warpgroups split every S row: wg 0 owns key columns [0, 64), wg 1
    // [64, 128) (and the same halves of O); the row max is combined through
    // smem with one named barrier per tile.  Two warps per SMSP hide the
    // LDTM / MUFU latencies one warpgroup alone exposes.
    const int q = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // row inside the tile == TMEM lane
    const int qi = q0 + r;        // query position inside the sequence
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    constexpr int HC = BN / 2;    // key columns per warpgroup
    constexpr int HD = D / 2;     // O columns per warpgroup
    const int c0 = wg * HC;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nt; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 32) tmem_ld_x32(tS[b] + lane_off + c0 + c, sv + c);
      tmem_ld_wait();
      // mask (only tiles touching the diagonal / sequence end; branch-free
      // select) + partial row max with 8 independent chains (raw scores)
      const int key0 = j * BN + c0;
      const bool need_mask = (j * BN + BN > kv_end) || (causal && j * BN + BN > q0);
      if (need_mask) {
        const int lim = causal ? min(S - key0, qi - key0 + 1) : (S - key0);  // keys [0, lim) valid
#pragma unroll
        for (int c = 0; c < HC; ++c) sv[c] = c < lim ? sv[c] : __float_as_uint(-INFINITY);
      }
      float pm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pm[i] = -INFINITY;
#pragma unroll
      for (int c = 0; c < HC; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sv[c]));
      const float mloc = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                               fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      red_max[j & 1][wg][r] = mloc;
      named_bar_sync(1, 256);  // both warpgroups of this tile
      const float mx = fmaxf(mloc, red_max[j & 1][wg ^ 1][r]) * scale_log2;
      float alpha = 1.f;
      if (mx > m_run + kRescaleThreshold || m_run == -INFINITY) {
        alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mx);
        m_run = mx;
        l_run *= alpha;
      }
      const float msub = (m_run == -INFINITY) ? 0.f : m_run;
      // P_j (bf16) overwrites this warpgroup's first 32 columns of its own S region
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[HC / 2];
#pragma unroll
      for (int c2 = 0; c2 < HC / 2; ++c2) {
        // p = 2^(s*scale_log2 - m); half the pairs on the SFU, half on the FMA pipe
        const float x0 = fmaf(__uint_as_float(sv[2 * c2]), scale_log2, -msub);
        const float x1 = fmaf(__uint_as_float(sv[2 * c2 + 1]), scale_log2, -msub);
        // (exp2_poly on the FMA pipe for half the pairs measured slower here: 459 vs 404 us)
        const float p0 = fast_exp2(x0);
        const float p1 = fast_exp2(x1);
        ls[c2 & 3] += p0 + p1;
        pk[c2] = pack_bf16x2(p0, p1);
      }
#pragma unroll
      for (int c = 0; c < HC / 2; c += 16) tmem_st_x16(tS[b] + lane_off + c0 + c, pk + c);
      l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      // rescale this warpgroup's half of O in TMEM when the running max moved
      const bool corr = (j > 0) && (alpha != 1.f);
      if (__any_sync(0xffffffffu, corr)) {
        mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
          uint32_t ov[32];
          tmem_ld_x32(tO + lane_off + wg * HD + c, ov);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st_x32(tO + lane_off + wg * HD + c, ov);
        }
        tmem_st_wait();
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[b]);
    }
    // epilogue: combine the two partial row sums, normalise this half of O
    red_max[nt & 1][wg][r] = l_run;  // parity nt&1 is no longer read by the loop
    mbar_wait(&o_final, 0);
    tc_fence_after();
    named_bar_sync(1, 256);
    const float l_tot = red_max[nt & 1][0][r] + red_max[nt & 1][1][r];
    const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
    __nv_bfloat16* orow = out + (int64_t)(tok0 + qi) * ldo + (int64_t)head * D + wg * HD;
#pragma unroll
    for (int c = 0; c < HD; c += 32) {
      uint32_t ov[32];
      tmem_ld_x32(tO + lane_off + wg * HD + c, ov);
      tmem_ld_wait();
      if (qi < S) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2)
            pk[k2] = pack_bf16x2(__uint_as_float(ov[i + 2 * k2]) * inv, __uint_as_float(ov[i + 2 * k2 + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + c + i) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
static int launch(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                  int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, float scale, int32_t causal,
                  cudaStream_t st) {
  const int64_t T = n_seqs * S;
  CUtensorMap mq, mk, mv;
  if (!encode_tmap_2d_bf16(&mq, q, (uint64_t)(n_q * D), (uint64_t)T, (uint64_t)ldq * 2, 64, BM, true) ||
      !encode_tmap_2d_bf16(&mk, k, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldk * 2, 64, BN, true) ||
      !encode_tmap_2d_bf16(&mv, v, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldv * 2, 64, BN, true))
    return HAP_ERR_DRIVER;
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)attn_tc_kernel<D>, Smem<D>::kTotal)) return HAP_ERR_LAUNCH;
    configured = 1;
  }
  dim3 grid((unsigned)((S + BM - 1) / BM), (unsigned)n_q, (unsigned)n_seqs);
  { if (hap::launch_k(attn_tc_kernel<D>, dim3(grid), dim3(kThreads), Smem<D>::kTotal, st, mq, mk, mv, reinterpret_cast<__nv_bfloat16*>(out), ldo,
                                                              (int)S, (int)n_q, (int)n_kv,
                                                              scale * 1.4426950408889634f, causal) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace attn_tc

// Entry used by hap_attn_prefill (attention.cu) for head_dim 64 / 128.
int attn_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                    int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, int64_t head_dim, float scale,
                    int32_t causal, cudaStream_t st) {
  if (head_dim == 128)
    return attn_tc::launch<128>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
  return attn_tc::launch<64>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
}

}  // namespace hap
