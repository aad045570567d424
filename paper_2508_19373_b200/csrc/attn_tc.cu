// Causal (or full) GQA prefill attention on 5th-gen tensor cores (tcgen05 +
// TMEM + TMA): a persistent two-Q-tile ping-pong kernel (FA4-style).
//
// Persistent: one CTA per SM fetches work items from a ticket counter in the
// caller's workspace (heaviest causal items first); the pipelines run across
// item boundaries, so the next item's Q load and first S = Q K^T overlap the
// current item's last softmax and its epilogue.  An item is a PAIR of 128-row
// Q tiles sharing one K/V stream (see attn_pair_kernel).  P is written back as
// bf16 over its own S columns in TMEM and is the TMEM A operand of the PV MMA
// (TS form); O is rescaled in TMEM only when the running max grows by > 2^8
// (exact: the same stale max is used for P and l).
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

// Work-item tickets: int32[2] in the caller's workspace (zero before the
// first launch).  The last CTA out of work re-zeroes them, so a workspace is
// reusable by the next launch on the same stream; concurrent launches need
// distinct workspaces.
constexpr size_t kSchedBytes = 2 * sizeof(int);

#define WAIT(b, p) mbar_wait_spin(b, p)
template <int D, int EMU>
__global__ void __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int64_t ldo, int S,
                     int n_q, int n_kv, int n_seqs, float scale_log2, int causal, int st32, int* __restrict__ sched,
                     int opt) {
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

  // registers: the role warpgroup (warps 0-3) runs scalar loops; each softmax
  // thread holds a 128-key S row plus its packed P (96*128 + 200*256 <= the
  // 168*384 the launch reserves)
  if (warp < 4) {
  setmaxnreg_dec<96>();
  if (warp == 0) {
    // ============ scheduler + Q loads ============
    if (lane == 0) {
      auto fetch = [&]() {
        const int v = atomicAdd(&sched[0], 1);
        return v < n_items ? v : -1;
      };
      int qc[2] = {0, 0};
      int cur = fetch();
      for (int ii = 0;; ++ii) {
        item_ring[ii & 7] = cur;
        mbar_arrive(&item_full[ii & 7]);
        if (cur < 0) {
          // the last CTA out of work leaves the scheduler zeroed for the next launch
          if (atomicAdd(&sched[1], 1) == (int)gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
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
  } else {
    // ============ MMA issuer (warp 1) ============
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
  }
  } else {
    setmaxnreg_inc<200>();
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
        // P = 2^(s*scale - m) into TMEM over S (bf16 pairs) and the row sum, in
        // packed fp32 pairs (FFMA2/FADD2); with EMU a fraction of the pairs takes
        // 2^x on the FMA pipe (exp2_poly2).  track: also reduce the raw row max.
        float pm[4];
        auto pass = [&](float msub, bool track) -> float {
          const uint64_t sc2 = f2dup(scale_log2), nm2 = f2dup(-msub);
          uint64_t ls2[2] = {0ull, 0ull};
#pragma unroll
          for (int i = 0; i < 4; ++i) pm[i] = -INFINITY;
#pragma unroll
          for (int h = 0; h < BN / 64; ++h) {
            uint32_t pk[32];
#pragma unroll
            for (int c2 = 0; c2 < 32; ++c2) {
              const float s0 = __uint_as_float(sv[64 * h + 2 * c2]), s1 = __uint_as_float(sv[64 * h + 2 * c2 + 1]);
              if (track) pm[c2 & 3] = fmaxf(pm[c2 & 3], fmaxf(s0, s1));
              const uint64_t x01 = ffma2r(f2pack(s0, s1), sc2, nm2);
              uint64_t p01;
              if ((EMU == 1 && (c2 & 3) == 3) || (EMU == 2 && (c2 & 7) == 7)) {
                p01 = exp2_poly2(x01);
              } else {
                const float2 xx = f2split(x01);
                p01 = f2pack(fast_exp2(xx.x), fast_exp2(xx.y));
              }
              fadd2(ls2[c2 & 1], p01);
              const float2 pp = f2split(p01);
              pk[c2] = pack_bf16x2(pp.x, pp.y);
            }
            tmem_st_x32(tS(t) + lane_off + 32 * h, pk);
          }
          const float2 a0 = f2split(ls2[0]), a1 = f2split(ls2[1]);
          return (a0.x + a0.y) + (a1.x + a1.y);
        };
        float alpha = 1.f;
        float lsum;
        if (opt && m_run != -INFINITY) {
          // optimistic: exponentials against the running max while the tile max
          // is reduced alongside (off the critical path); a row whose max grew
          // past the threshold redoes its pass with the new max — the same
          // values the max-first order produces
          lsum = pass(m_run, true);
          const float mx =
              fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])) * scale_log2;
          if (mx > m_run + kRescaleThreshold) {
            alpha = fast_exp2(m_run - mx);
            m_run = mx;
            l_run *= alpha;
            lsum = pass(m_run, false);
          }
        } else {
          float pq[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) pq[i] = __uint_as_float(sv[i]);
#pragma unroll
          for (int c = 8; c < BN; ++c) pq[c & 7] = fmaxf(pq[c & 7], __uint_as_float(sv[c]));
          const float mx = fmaxf(fmaxf(fmaxf(pq[0], pq[1]), fmaxf(pq[2], pq[3])),
                                 fmaxf(fmaxf(pq[4], pq[5]), fmaxf(pq[6], pq[7]))) *
                           scale_log2;
          if (mx > m_run + kRescaleThreshold || m_run == -INFINITY) {
            alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mx);
            m_run = mx;
            l_run *= alpha;
          }
          lsum = pass((m_run == -INFINITY) ? 0.f : m_run, false);
        }
        l_run += lsum;
        // PV_t,j-1 has landed (S_t,j, already in TMEM, was issued after it);
        // every o_done phase is waited so the barrier protocol stays explicit
        if (j > 0) WAIT(&o_done[t], (sc - 1) & 1);
        // rescale O in TMEM when the running max moved
        if (__any_sync(0xffffffffu, j > 0 && alpha != 1.f)) {
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
      WAIT(&o_done[t], (sc - 1) & 1);  // the item's last PV (same completion as o_final)
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

static int attn_opt() {
  static const int on = [] {
    // A/B switch, default off: exponentials against the running max with the
    // tile max reduced alongside (+ a redo for rows whose max moved) measured
    // bit-identical and no faster (causal 328-329 vs 325-327 us): the softmax
    // is bound by the SFU and issue slots, not by the max's latency
    const char* e = getenv("HAP_ATTN_OPT");
    return e ? atoi(e) : 0;
  }();
  return on;
}

template <int D, int EMU>
static int launch_pair(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                       int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, float scale, int32_t causal,
                       int* sched, cudaStream_t st) {
  const int64_t T = n_seqs * S;
  CUtensorMap mq, mk, mv;
  if (!encode_tmap_2d_bf16(&mq, q, (uint64_t)(n_q * D), (uint64_t)T, (uint64_t)ldq * 2, 64, BM, true) ||
      !encode_tmap_2d_bf16(&mk, k, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldk * 2, 64, BN, true) ||
      !encode_tmap_2d_bf16(&mv, v, (uint64_t)(n_kv * D), (uint64_t)T, (uint64_t)ldv * 2, 64, BN, true))
    return HAP_ERR_DRIVER;
  auto kern = attn_pair_kernel<D, EMU>;
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
                    (int)(((reinterpret_cast<uintptr_t>(out) | (uintptr_t)(ldo * 2)) & 31) == 0), sched,
                    attn_opt()) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace attn_tc

size_t attn_prefill_tc_workspace_bytes() { return attn_tc::kSchedBytes; }

// Entry used by hap_attn_prefill (attention.cu) for head_dim 64 / 128.
int attn_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* out,
                    int64_t ldo, int64_t n_seqs, int64_t S, int64_t n_q, int64_t n_kv, int64_t head_dim, float scale,
                    int32_t causal, int* sched, cudaStream_t st) {
  static int emu = -1;
  if (emu < 0) {
    // A/B switch: 0 = every exponential on the SFU (default, measured fastest:
    // causal 316-318 us vs 340-343 us with one pair in four on the FMA pipe),
    // 1 = one exp2 pair in four / 2 = one in eight through exp2_poly2
    const char* e = getenv("HAP_ATTN_EMU");
    emu = e ? atoi(e) : 0;
  }
#define HAP_ATTN_CASE(DD, EE)                                                                                    \
  if (head_dim == DD && emu == EE)                                                                               \
    return attn_tc::launch_pair<DD, EE>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, \
                                        sched, st);
  HAP_ATTN_CASE(128, 1)
  HAP_ATTN_CASE(128, 2)
  HAP_ATTN_CASE(64, 1)
  HAP_ATTN_CASE(64, 2)
#undef HAP_ATTN_CASE
  if (head_dim == 128)
    return attn_tc::launch_pair<128, 0>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, sched,
                                        st);
  return attn_tc::launch_pair<64, 0>(q, ldq, k, ldk, v, ldv, out, ldo, n_seqs, S, n_q, n_kv, scale, causal, sched,
                                     st);
}

}  // namespace hap
