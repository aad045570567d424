// Causal GQA prefill attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Persistent: one CTA per SM walks work items (128-query tile, q head,
// sequence), heaviest causal tiles first, round-robin over the grid.  The
// pipelines run across item boundaries, so the next item's Q load and first
// S = Q K^T MMA overlap the current item's last softmax and its epilogue (a
// one-CTA-per-item launch paid ~5.8 us of fill/drain per item).  12 warps:
//   warp 0      TMA producer: Q (double-buffered per item), then the K ring
//   warp 3      TMA producer: the V ring
//   warp 1      MMA issuer (one thread): S_j into a double-buffered TMEM S
//               tile (128x128 fp32); O += P_{j-1} V_{j-1} into the item's TMEM
//               O buffer (two O buffers alternate between items), so S_{j+1}
//               overlaps the softmax of tile j and PV_j the softmax of j+1
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4..11 softmax + epilogue, two warpgroups splitting each row: thread
//               = one query row (its TMEM lane); tcgen05.ld the S row, causal
//               mask, exp2-domain online softmax with a lazily updated running
//               max (O is rescaled in TMEM only when the max grows by > 2^8 —
//               exact, as the same stale max is used for P and l); P is written
//               back as bf16 over its own S columns (TS-form PV MMA reads it
//               from TMEM)
// Final per item: O row / l -> bf16 -> global, then the O buffer is released.
//
// Models: score+value term 4*n*kv_len*h of attention_flops (reference
// arch.py:161); causal: tiles above the diagonal are skipped.
#include <cstdlib>

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
  static constexpr int kTotal = 2 * kQ + 2 * kK + 2 * kV + 1024;  // P lives in TMEM
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

struct AttnItem {
  int mb, head, seq, kvh, q0, tok0, kv_end, nt;
};

__device__ __forceinline__ AttnItem attn_item(int it, int S, int n_q, int n_kv, int n_seqs, int causal) {
  // q-tiles of one (head, sequence) are consecutive, longest causal rows first:
  // concurrently running items share K/V in L2, and the tail of the dynamic
  // schedule is made of the shortest rows
  AttnItem a;
  const int n_mblk = (S + BM - 1) / BM;
  const int m = it % n_mblk, hs = it / n_mblk;
  a.mb = causal ? (n_mblk - 1 - m) : m;
  a.head = hs % n_q;
  a.seq = hs / n_q;
  a.kvh = a.head / (n_q / n_kv);
  a.q0 = a.mb * BM;
  a.tok0 = a.seq * S;
  a.kv_end = causal ? min(S, a.q0 + BM) : S;
  a.nt = (a.kv_end + BN - 1) / BN;
  return a;
}

// Dynamic item scheduler: items are numbered by decreasing cost (causal rows
// longest first) and fetched with an atomic ticket by each CTA's Q producer,
// which forwards them to the other roles through an 8-slot smem ring (the
// producer runs at most ~3 items ahead of the slowest reader).  The last CTA
// to run out of work re-zeroes the tickets, so the kernel leaves them ready for
// the next launch on the stream (launches of this kernel must not run
// concurrently on several streams of one device).
__device__ int g_attn_sched[2];

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int64_t ldo, int S,
                   int n_q, int n_kv, int n_seqs, float scale_log2, int causal) {
  pdl_trigger();
  pdl_wait();
  using SM = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sQ = smem;                  // [2][kQ]
  uint8_t* sK = sQ + 2 * SM::kQ;       // [2][kK]
  uint8_t* sV = sK + 2 * SM::kK;       // [2][kV]

  __shared__ __align__(8) uint64_t q_full[2], q_empty[2];
  __shared__ __align__(8) uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  __shared__ __align__(8) uint64_t s_full[2], p_full[2], o_done[2];
  __shared__ __align__(8) uint64_t o_final[2], o_free[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ float red_max[2][2][BM];  // [tile parity][warpgroup][row]
  __shared__ float red_l[2][BM];       // [warpgroup][row], item epilogue
  __shared__ int item_ring[8];
  __shared__ __align__(8) uint64_t item_full[8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = ((S + BM - 1) / BM) * n_q * n_seqs;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 256);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_final[i], 1);
      mbar_init(&o_free[i], 256);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&item_full[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&tmem_base_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tOb[2] = {tmem + 256, tmem + 384};

  if (warp == 0) {
    // ===================== TMA producer: Q per item, then the K ring =====================
    // K_j is consumed by S_j only, so its stage is released as soon as S_j
    // completes and K runs ahead of V (separate ring, separate thread).
    if (lane == 0) {
      int kc = 0;
      for (int ii = 0;; ++ii) {
        const int v = atomicAdd(&g_attn_sched[0], 1);
        const int it = v < n_items ? v : -1;
        item_ring[ii & 7] = it;
        mbar_arrive(&item_full[ii & 7]);
        if (it < 0) {
          // the last CTA out of work leaves the scheduler zeroed for the next launch
          if (atomicAdd(&g_attn_sched[1], 1) == (int)gridDim.x - 1) {
            g_attn_sched[0] = 0;
            g_attn_sched[1] = 0;
          }
          break;
        }
        const AttnItem a = attn_item(it, S, n_q, n_kv, n_seqs, causal);
        const int qb = ii & 1;
        mbar_wait(&q_empty[qb], ((ii >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], SM::kQ);
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(sQ + qb * SM::kQ + c * kChunkBytes, &tmQ, &q_full[qb], a.head * D + c * 64, a.tok0 + a.q0,
                      kEvictFirst);
        for (int j = 0; j < a.nt; ++j, ++kc) {
          const int s = kc & 1;
          mbar_wait(&k_empty[s], ((kc >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[s], SM::kK);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(sK + s * SM::kK + c * kChunkBytes, &tmK, &k_full[s], a.kvh * D + c * 64, a.tok0 + j * BN,
                        kEvictLast);
        }
      }
    }
  } else if (warp == 3) {
    // ===================== TMA producer: the V ring (released after PV_j) =====================
    if (lane == 0) {
      int vc = 0;
      for (int ii = 0;; ++ii) {
        mbar_wait(&item_full[ii & 7], (ii >> 3) & 1);
        const int it = item_ring[ii & 7];
        if (it < 0) break;
        const AttnItem a = attn_item(it, S, n_q, n_kv, n_seqs, causal);
        for (int j = 0; j < a.nt; ++j, ++vc) {
          const int s = vc & 1;
          mbar_wait(&v_empty[s], ((vc >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[s], SM::kV);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(sV + s * SM::kV + c * kChunkBytes, &tmV, &v_full[s], a.kvh * D + c * 64, a.tok0 + j * BN,
                        kEvictLast);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idS = make_idesc_bf16(BM, BN);
      const uint32_t idPV = make_idesc_bf16(BM, D) | (1u << 16);  // B (V) is MN-major
      // PV of tile tcp (index jp inside its item) into O buffer ob; the last
      // tile of an item also commits o_final[ob]
      auto issue_pv = [&](int tcp, int jp, int ob, bool last) {
        const int bp = tcp & 1;
        mbar_wait(&v_full[bp], (tcp >> 1) & 1);
        mbar_wait(&p_full[bp], (tcp >> 1) & 1);
        tc_fence_after();
        const uint32_t vbase = smem_u32(sV + bp * SM::kV);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // P sits in its S buffer: warpgroup w's 64 keys packed into columns [w*64, w*64+32)
          const uint32_t ta = tS[bp] + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint64_t db = make_sdesc_mn_sw128(vbase + kk * 16 * 128, kChunkBytes);
          umma_bf16_ts(tOb[ob], ta, db, idPV, (jp | kk) != 0);
        }
        umma_commit(&o_done[bp]);
        umma_commit(&v_empty[bp]);
        if (last) umma_commit(&o_final[ob]);
      };
      // PV_j is issued after S_{j+1} (the next item's S_0 for an item's last
      // tile); the first PV into an O buffer waits for the epilogue of the item
      // two back to release it (o_free[ob] completes once per item)
      int tc = 0;
      int pend_tc = -1, pend_j = 0, pend_ii = 0;
      bool pend_last = false;
      auto issue_pend = [&]() {
        const int pob = pend_ii & 1;
        if (pend_j == 0) mbar_wait(&o_free[pob], ((pend_ii >> 1) & 1) ^ 1);
        tc_fence_after();
        issue_pv(pend_tc, pend_j, pob, pend_last);
      };
      for (int ii = 0;; ++ii) {
        mbar_wait(&item_full[ii & 7], (ii >> 3) & 1);
        const int it = item_ring[ii & 7];
        if (it < 0) break;
        const AttnItem a = attn_item(it, S, n_q, n_kv, n_seqs, causal);
        const int qb = ii & 1;
        mbar_wait(&q_full[qb], (ii >> 1) & 1);
        const uint32_t qbase = smem_u32(sQ + qb * SM::kQ);
        for (int j = 0; j < a.nt; ++j, ++tc) {
          const int s = tc & 1;
          mbar_wait(&k_full[s], (tc >> 1) & 1);
          tc_fence_after();
          const uint32_t kbase = smem_u32(sK + s * SM::kK);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t da = make_sdesc_sw128(qbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
            const uint64_t db = make_sdesc_sw128(kbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
            umma_bf16_ss(tS[s], da, db, idS, kk != 0);
          }
          umma_commit(&s_full[s]);
          umma_commit(&k_empty[s]);
          if (j == a.nt - 1) umma_commit(&q_empty[qb]);  // last read of this item's Q
          if (pend_tc >= 0) issue_pend();
          pend_tc = tc;
          pend_j = j;
          pend_ii = ii;
          pend_last = j == a.nt - 1;
        }
      }
      if (pend_tc >= 0) issue_pend();
    }
  } else if (warp >= 4) {
    // ===================== softmax + epilogue =====================
    // Two warpgroups split every S row: wg 0 owns key columns [0, 64), wg 1
    // [64, 128) (and the same halves of O); the row max is combined through
    // smem with one named barrier per tile.
    const int q = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // row inside the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    constexpr int HC = BN / 2;    // key columns per warpgroup
    constexpr int HD = D / 2;     // O columns per warpgroup
    const int c0 = wg * HC;
    // item epilogue: combine the two partial row sums, normalise this half of O,
    // store, release the O buffer to the MMA (item ii + 2 reuses it)
    auto epilogue = [&](int eii, const AttnItem& ea, float el) {
      const int ob = eii & 1;
      const int qi = ea.q0 + r;
      red_l[wg][r] = el;
      mbar_wait(&o_final[ob], (eii >> 1) & 1);
      tc_fence_after();
      named_bar_sync(1, 256);
      const float l_tot = red_l[0][r] + red_l[1][r];
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
      __nv_bfloat16* orow = out + (int64_t)(ea.tok0 + qi) * ldo + (int64_t)ea.head * D + wg * HD;
#pragma unroll
      for (int c = 0; c < HD; c += 32) {
        uint32_t ov[32];
        tmem_ld_x32(tOb[ob] + lane_off + wg * HD + c, ov);
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
      tc_fence_before();
      mbar_arrive(&o_free[ob]);
    };
    int pend_ii = -1;
    AttnItem pend_a{};
    float pend_l = 0.f;
    int tc = 0;
    for (int ii = 0;; ++ii) {
        mbar_wait(&item_full[ii & 7], (ii >> 3) & 1);
        const int it = item_ring[ii & 7];
        if (it < 0) break;
      const AttnItem a = attn_item(it, S, n_q, n_kv, n_seqs, causal);
      const int ob = ii & 1;
      const int qi = a.q0 + r;  // query position inside the sequence
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < a.nt; ++j, ++tc) {
        const int b = tc & 1;
        mbar_wait(&s_full[b], (tc >> 1) & 1);
        tc_fence_after();
        uint32_t sv[HC];
#pragma unroll
        for (int c = 0; c < HC; c += 32) tmem_ld_x32(tS[b] + lane_off + c0 + c, sv + c);
        tmem_ld_wait();
        // mask (only tiles touching the diagonal / sequence end; branch-free
        // select) + partial row max with 8 independent chains (raw scores)
        const int key0 = j * BN + c0;
        const bool need_mask = (j * BN + BN > a.kv_end) || (causal && j * BN + BN > a.q0);
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
        red_max[b][wg][r] = mloc;
        named_bar_sync(1, 256);  // both warpgroups of this tile
        const float mx = fmaxf(mloc, red_max[b][wg ^ 1][r]) * scale_log2;
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
          const float x0 = fmaf(__uint_as_float(sv[2 * c2]), scale_log2, -msub);
          const float x1 = fmaf(__uint_as_float(sv[2 * c2 + 1]), scale_log2, -msub);
          // (a degree-3 FMA-pipe exp2 for 1/8..3/8 of the pairs measured 3-12 % slower)
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
          mbar_wait(&o_done[(tc - 1) & 1], ((tc - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD; c += 32) {
            uint32_t ov[32];
            tmem_ld_x32(tOb[ob] + lane_off + wg * HD + c, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_x32(tOb[ob] + lane_off + wg * HD + c, ov);
          }
          tmem_st_wait();
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[b]);
      }
      // the epilogue of the previous item runs now, one item late: its last PV
      // (issued behind this item's S_0) finished long ago, so the softmax warps
      // never idle on o_final; O is double-buffered, so this item's PVs are
      // unaffected
      if (pend_ii >= 0) epilogue(pend_ii, pend_a, pend_l);
      pend_ii = ii;
      pend_a = a;
      pend_l = l_run;
    }
    if (pend_ii >= 0) epilogue(pend_ii, pend_a, pend_l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// ============================================================================
// Two-tile ping-pong kernel (the default).  A work item is a PAIR of 128-row
// Q tiles sharing one K/V stream: two heads of one GQA group at the same rows
// when the group size is even, else two consecutive q-tiles of one head (the
// lower tile needs one causal K/V tile fewer).  Softmax warpgroup t owns Q
// tile t with one thread per full 128-key row (no cross-warpgroup max
// exchange), and the MMA issuer alternates [PV_a,j-1  S_a,j] [PV_b,j-1  S_b,j]:
// while one warpgroup runs its (SFU-bound) softmax the tensor pipe works on
// the other tile.  TMEM: S_a | S_b | O_a | O_b; P_t (bf16) overwrites the
// first 64 columns of S_t and is the TMEM A operand of PV_t.
// Roles: warp 0 scheduler + Q loads (per-tile buffers; the next item's Q is
// prefetched into L2 when the current one starts), warp 1 MMA issuer, warp 2
// TMEM allocator + K ring, warp 3 V ring, warps 4-7 / 8-11 softmax and
// epilogue of tile a / b.
// ============================================================================
// 2^x on the FMA pipe (x <= 0): round-to-nearest split x = n + f via the
// 1.5*2^23 magic constant, degree-3 minimax polynomial for 2^f on [-0.5, 0.5]
// (max relative error 7.5e-5, far below the bf16 rounding of P), n added to
// the exponent field.  Offloads part of the exponentials from the SFU, which
// otherwise takes as long per tile pair as the tensor pipe.
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float j = x + 12582912.f;
  const float f = x - (j - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517177f, f, 0.24261138f), f, 0.69326097f), f, 0.999928f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

template <int D>
struct PairSmem {
  static constexpr int kTile = (D / 64) * kChunkBytes;  // one 128-row operand tile
  static constexpr int kKS = D == 128 ? 2 : 4;           // K ring stages
  static constexpr int kVS = D == 128 ? 2 : 4;           // V ring stages (V_j is held until PV_b,j)
  static constexpr int kTotal = (2 + kKS + kVS) * kTile + 1024;  // Q_a, Q_b, K ring, V ring
};

struct PairTile {
  int head, q0, kv_end, nt;
};
struct PairItem {
  PairTile t[2];  // t[0].nt <= t[1].nt; t[0].nt == 0 when the item holds one tile
  int kvh, tok0;
};

__device__ __forceinline__ PairItem pair_item(int it, int S, int n_q, int n_kv, int causal) {
  PairItem a;
  const int n_mblk = (S + BM - 1) / BM;
  const int G = n_q / n_kv;
  auto mk = [&](int head, int mb) {
    PairTile t;
    t.head = head;
    t.q0 = mb * BM;
    t.kv_end = causal ? min(S, t.q0 + BM) : S;
    t.nt = (t.kv_end + BN - 1) / BN;
    return t;
  };
  int seq;
  if ((G & 1) == 0) {
    // heads (2p, 2p+1) of one KV group at q-tile m, longest causal rows first
    const int n_hp = n_q / 2;
    const int m = it % n_mblk, rest = it / n_mblk;
    const int mb = causal ? n_mblk - 1 - m : m;
    const int hp = rest % n_hp;
    seq = rest / n_hp;
    a.t[0] = mk(2 * hp, mb);
    a.t[1] = mk(2 * hp + 1, mb);
  } else {
    // q-tiles (2p, 2p+1) of one head
    const int n_mp = (n_mblk + 1) / 2;
    const int m = it % n_mp, rest = it / n_mp;
    const int mp = causal ? n_mp - 1 - m : m;
    const int head = rest % n_q;
    seq = rest / n_q;
    if (2 * mp + 1 < n_mblk) {
      a.t[0] = mk(head, 2 * mp);
      a.t[1] = mk(head, 2 * mp + 1);
    } else {
      a.t[1] = mk(head, 2 * mp);
      a.t[0] = a.t[1];
      a.t[0].nt = 0;
    }
  }
  a.kvh = a.t[1].head / G;
  a.tok0 = seq * S;
  return a;
}

__device__ __forceinline__ int pair_items(int S, int n_q, int n_kv, int n_seqs) {
  const int n_mblk = (S + BM - 1) / BM;
  return ((n_q / n_kv) & 1) == 0 ? n_mblk * (n_q / 2) * n_seqs : ((n_mblk + 1) / 2) * n_q * n_seqs;
}

__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

__device__ int g_attn_pair_sched[2];


#define WAIT(b, p) (kSpin ? mbar_wait_spin(b, p) : mbar_wait(b, p))
template <int D, int kPoly, bool kSpin = true>  // kPoly of every 8 exp2 pairs on the FMA pipe
__global__ void __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int64_t ldo, int S,
                     int n_q, int n_kv, int n_seqs, float scale_log2, int causal, int st32) {
  pdl_trigger();
  pdl_wait();
  constexpr int kTile = PairSmem<D>::kTile;
  constexpr int kKS = PairSmem<D>::kKS, kVS = PairSmem<D>::kVS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sQ = smem;            // [tile][kTile]
  uint8_t* sK = sQ + 2 * kTile;  // [stage][kTile]
  uint8_t* sV = sK + kKS * kTile;  // [stage][kTile]

  __shared__ __align__(8) uint64_t q_full[2], q_empty[2];
  __shared__ __align__(8) uint64_t k_full[kKS], k_empty[kKS], v_full[kVS], v_empty[kVS];
  __shared__ __align__(8) uint64_t s_full[2], p_full[2], o_done[2], o_final[2], o_free[2];
  __shared__ __align__(8) uint64_t item_full[8];
  __shared__ int item_ring[8];
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = pair_items(S, n_q, n_kv, n_seqs);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_final[i], 1);
      mbar_init(&o_free[i], 128);
    }
    for (int i = 0; i < kKS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&item_full[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&tmem_base_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  auto tS = [&](int t) { return tmem + 128u * t; };
  auto tO = [&](int t) { return tmem + 256u + (uint32_t)D * t; };

  if (warp == 0) {
    // ============ scheduler + Q loads ============
    if (lane == 0) {
      auto fetch = [&]() {
        const int v = atomicAdd(&g_attn_pair_sched[0], 1);
        return v < n_items ? v : -1;
      };
      int qc[2] = {0, 0};
      int cur = fetch();
      for (int ii = 0;; ++ii) {
        item_ring[ii & 7] = cur;
        mbar_arrive(&item_full[ii & 7]);
        if (cur < 0) {
          // the last CTA out of work leaves the scheduler zeroed for the next launch
          if (atomicAdd(&g_attn_pair_sched[1], 1) == (int)gridDim.x - 1) {
            g_attn_pair_sched[0] = 0;
            g_attn_pair_sched[1] = 0;
          }
          break;
        }
        const int nxt = fetch();
        if (nxt >= 0) {
          const PairItem b = pair_item(nxt, S, n_q, n_kv, causal);
          for (int t = 0; t < 2; ++t)
            if (b.t[t].nt > 0)
              for (int c = 0; c < D / 64; ++c) tma_prefetch_l2_2d(&tmQ, b.t[t].head * D + c * 64, b.tok0 + b.t[t].q0);
        }
        const PairItem a = pair_item(cur, S, n_q, n_kv, causal);
        for (int t = 0; t < 2; ++t) {
          if (a.t[t].nt == 0) continue;
          WAIT(&q_empty[t], (qc[t] & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[t], kTile);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(sQ + t * kTile + c * kChunkBytes, &tmQ, &q_full[t], a.t[t].head * D + c * 64,
                        a.tok0 + a.t[t].q0, kEvictFirst);
          ++qc[t];
        }
        cur = nxt;
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ============ K ring (warp 2, after the TMEM allocation) / V ring (warp 3) ============
    if (lane == 0) {
      const bool isK = warp == 2;
      const CUtensorMap* map = isK ? &tmK : &tmV;
      uint8_t* ring = isK ? sK : sV;
      uint64_t* full = isK ? k_full : v_full;
      uint64_t* empty = isK ? k_empty : v_empty;
      const int nst = isK ? kKS : kVS;
      int c = 0;
      for (int ii = 0;; ++ii) {
        WAIT(&item_full[ii & 7], (ii >> 3) & 1);
        const int it = item_ring[ii & 7];
        if (it < 0) break;
        const PairItem a = pair_item(it, S, n_q, n_kv, causal);
        for (int j = 0; j < a.t[1].nt; ++j, ++c) {
          const int st = c % nst;
          WAIT(&empty[st], ((c / nst) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], kTile);
          for (int cc = 0; cc < D / 64; ++cc)
            tma_load_2d(ring + st * kTile + cc * kChunkBytes, map, &full[st], a.kvh * D + cc * 64, a.tok0 + j * BN,
                        kEvictLast);
        }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer ============
    // Per K/V step j: [PV_a,j-1  S_a,j] [PV_b,j-1  S_b,j].  S_t,j overwrites
    // P_t,j-1, so it is issued behind PV_t,j-1 (tcgen05 ops of one thread run
    // in order); the PVs of an item's last step are issued at the next item's
    // first step.  One issuer keeps the two softmax warpgroups half a period
    // apart (a per-tile issuer was measured 38 % slower: the softmaxes fell
    // into phase and shared the SFU).
    if (lane == 0) {
      const uint32_t idS = make_idesc_bf16(BM, BN);
      const uint32_t idPV = make_idesc_bf16(BM, D) | (1u << 16);  // B (V) is MN-major
      struct Pend {
        int valid, j, last, kv, item;  // kv: global K/V tile index, item: per-tile item count
      };
      Pend pend[2] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
      int pc[2] = {0, 0};  // PVs issued per tile (p_full phase)
      int qc[2] = {0, 0};  // Q loads consumed per tile
      int ic[2] = {0, 0};  // items per tile (o_free phase)
      auto issue_pv = [&](int t) {
        const Pend& p = pend[t];
        const int vs = p.kv % kVS;
        WAIT(&v_full[vs], (p.kv / kVS) & 1);
        WAIT(&p_full[t], pc[t] & 1);
        ++pc[t];
        if (p.j == 0) WAIT(&o_free[t], (p.item & 1) ^ 1);  // epilogue of this tile's previous item
        tc_fence_after();
        const uint32_t vbase = smem_u32(sV + vs * kTile);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t db = make_sdesc_mn_sw128(vbase + kk * 16 * 128, kChunkBytes);
          umma_bf16_ts(tO(t), tS(t) + kk * 8, db, idPV, (p.j | kk) != 0);
        }
        umma_commit(&o_done[t]);
        if (t == 1) umma_commit(&v_empty[vs]);  // PV_b,j is the last reader of V_j
        if (p.last) umma_commit(&o_final[t]);
        pend[t].valid = 0;
      };
      int kc = 0;
      for (int ii = 0;; ++ii) {
        WAIT(&item_full[ii & 7], (ii >> 3) & 1);
        const int it = item_ring[ii & 7];
        if (it < 0) break;
        const PairItem a = pair_item(it, S, n_q, n_kv, causal);
        const int nt_b = a.t[1].nt;
        for (int j = 0; j < nt_b; ++j, ++kc) {
          const int ks = kc % kKS;
          bool k_ready = false;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (pend[t].valid) issue_pv(t);
            if (j >= a.t[t].nt) continue;
            if (j == 0) {
              WAIT(&q_full[t], qc[t] & 1);
              ++qc[t];
            }
            if (!k_ready) {
              WAIT(&k_full[ks], (kc / kKS) & 1);
              k_ready = true;
            }
            tc_fence_after();
            const uint32_t qbase = smem_u32(sQ + t * kTile);
            const uint32_t kbase = smem_u32(sK + ks * kTile);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t da = make_sdesc_sw128(qbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
              const uint64_t db = make_sdesc_sw128(kbase + (kk >> 2) * kChunkBytes) + 2 * (kk & 3);
              umma_bf16_ss(tS(t), da, db, idS, kk != 0);
            }
            umma_commit(&s_full[t]);
            const bool last = j == a.t[t].nt - 1;
            if (last) umma_commit(&q_empty[t]);
            pend[t] = {1, j, last ? 1 : 0, kc, ic[t]};
          }
          umma_commit(&k_empty[ks]);
        }
        if (a.t[0].nt > 0) ++ic[0];
        ++ic[1];
      }
      if (pend[0].valid) issue_pv(0);
      if (pend[1].valid) issue_pv(1);
    }
  } else if (warp >= 4) {
    // ============ softmax + epilogue, warpgroup t owns Q tile t ============
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;  // row inside the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int sc = 0;  // S tiles consumed (s_full / o_done phase)
    int ic = 0;  // items of this tile (o_final phase)
    for (int ii = 0;; ++ii) {
      WAIT(&item_full[ii & 7], (ii >> 3) & 1);
      const int it = item_ring[ii & 7];
      if (it < 0) break;
      const PairItem a = pair_item(it, S, n_q, n_kv, causal);
      const PairTile tl = a.t[t];
      if (tl.nt == 0) continue;
      const int qi = tl.q0 + r;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < tl.nt; ++j, ++sc) {
        WAIT(&s_full[t], sc & 1);
        tc_fence_after();
        uint32_t sv[BN];
#pragma unroll
        for (int c = 0; c < BN; c += 32) tmem_ld_x32(tS(t) + lane_off + c, sv + c);
        tmem_ld_wait();
        const int key0 = j * BN;
        if (key0 + BN > tl.kv_end || (causal && key0 + BN > tl.q0)) {
          const int lim = causal ? min(S - key0, qi - key0 + 1) : (S - key0);  // keys [0, lim) valid
#pragma unroll
          for (int c = 0; c < BN; ++c) sv[c] = c < lim ? sv[c] : __float_as_uint(-INFINITY);
        }
        float pm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pm[i] = __uint_as_float(sv[i]);
#pragma unroll
        for (int c = 8; c < BN; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sv[c]));
        const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                               fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) *
                         scale_log2;
        float alpha = 1.f;
        if (mx > m_run + kRescaleThreshold || m_run == -INFINITY) {
          alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mx);
          m_run = mx;
          l_run *= alpha;
        }
        const float msub = (m_run == -INFINITY) ? 0.f : m_run;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int h = 0; h < BN / 64; ++h) {
          uint32_t pk[32];
#pragma unroll
          for (int c2 = 0; c2 < 32; ++c2) {
            const float x0 = fmaf(__uint_as_float(sv[64 * h + 2 * c2]), scale_log2, -msub);
            const float x1 = fmaf(__uint_as_float(sv[64 * h + 2 * c2 + 1]), scale_log2, -msub);
            const bool poly = (c2 & 7) < kPoly;
            const float p0 = poly ? exp2_fma(x0) : fast_exp2(x0);
            const float p1 = poly ? exp2_fma(x1) : fast_exp2(x1);
            ls[c2 & 3] += p0 + p1;
            pk[c2] = pack_bf16x2(p0, p1);
          }
          tmem_st_x32(tS(t) + lane_off + 32 * h, pk);
        }
        l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        // rescale O in TMEM when the running max moved (PV_t,j-1 must have landed)
        if (__any_sync(0xffffffffu, j > 0 && alpha != 1.f)) {
          WAIT(&o_done[t], (sc - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            uint32_t ov[32];
            tmem_ld_x32(tO(t) + lane_off + c, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_x32(tO(t) + lane_off + c, ov);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[t]);  // per-thread arrive (a warp-level arrive was measured slower)
      }
      // epilogue: O row / l -> bf16 -> global, then release O_t
      WAIT(&o_final[t], ic & 1);
      ++ic;
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow = out + (int64_t)(a.tok0 + qi) * ldo + (int64_t)tl.head * D;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t ov[32];
        tmem_ld_x32(tO(t) + lane_off + c, ov);
        tmem_ld_wait();
        if (qi < S) {
          if (st32) {
#pragma unroll
            for (int i = 0; i < 32; i += 16) {
              uint32_t pk[8];
#pragma unroll
              for (int k2 = 0; k2 < 8; ++k2)
                pk[k2] = pack_bf16x2(__uint_as_float(ov[i + 2 * k2]) * inv, __uint_as_float(ov[i + 2 * k2 + 1]) * inv);
              st_global_v8(orow + c + i, pk);
            }
          } else {
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
      mbar_arrive(&o_free[t]);
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
static int launch_pair(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                       int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, float scale, int32_t causal,
                       cudaStream_t st) {
  const int64_t T = n_seqs * S;
  CUtensorMap mq, mk, mv;
  if (!encode_tmap_2d_bf16(&mq, q, (uint64_t)(n_q * D), (uint64_t)T, (uint64_t)ldq * 2, 64, BM, true) ||
      !encode_tmap_2d_bf16(&mk, k, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldk * 2, 64, BN, true) ||
      !encode_tmap_2d_bf16(&mv, v, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldv * 2, 64, BN, true))
    return HAP_ERR_DRIVER;
  static const int variant = [] {
    const char* e = getenv("HAP_ATTN_VARIANT");  // tuning experiments only: bit 0 poly, bit 1 suspend-hint waits
    return e ? atoi(e) & 3 : 0;
  }();
  auto kern = variant == 0 ? attn_pair_kernel<D, 0, true>
                           : variant == 1 ? attn_pair_kernel<D, 1, true>
                                          : variant == 2 ? attn_pair_kernel<D, 0, false> : attn_pair_kernel<D, 1, false>;
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)kern, PairSmem<D>::kTotal)) return HAP_ERR_LAUNCH;
    configured = 1;
  }
  const int64_t n_mblk = (S + BM - 1) / BM;
  const int64_t n_items = ((n_q / n_kv) % 2 == 0) ? n_mblk * (n_q / 2) * n_seqs : ((n_mblk + 1) / 2) * n_q * n_seqs;
  const unsigned grid = (unsigned)(n_items < kNumSMs ? n_items : kNumSMs);
  if (hap::launch_k(kern, dim3(grid), dim3(kThreads), PairSmem<D>::kTotal, st, mq, mk, mv,
                    reinterpret_cast<__nv_bfloat16*>(out), ldo, (int)S, (int)n_q, (int)n_kv, (int)n_seqs,
                    scale * 1.4426950408889634f, causal,
                    (int)(((reinterpret_cast<uintptr_t>(out) | (uintptr_t)(ldo * 2)) & 31) == 0)) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
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
  const int64_t n_items = ((S + BM - 1) / BM) * n_q * n_seqs;
  const unsigned grid = (unsigned)(n_items < kNumSMs ? n_items : kNumSMs);
  { if (hap::launch_k(attn_tc_kernel<D>, dim3(grid), dim3(kThreads), Smem<D>::kTotal, st, mq, mk, mv, reinterpret_cast<__nv_bfloat16*>(out), ldo,
                                                              (int)S, (int)n_q, (int)n_kv, (int)n_seqs,
                                                              scale * 1.4426950408889634f, causal) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace attn_tc

// Entry used by hap_attn_prefill (attention.cu) for head_dim 64 / 128.
int attn_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                    int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, int64_t head_dim, float scale,
                    int32_t causal, cudaStream_t st) {
  static const int impl = [] {
    const char* e = getenv("HAP_ATTN_IMPL");  // A/B experiments only: 1 = single-tile kernel
    return e ? atoi(e) : 0;
  }();
  if (impl == 1) {
    if (head_dim == 128)
      return attn_tc::launch<128>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
    return attn_tc::launch<64>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
  }
  if (head_dim == 128)
    return attn_tc::launch_pair<128>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
  return attn_tc::launch_pair<64>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, st);
}

}  // namespace hap
