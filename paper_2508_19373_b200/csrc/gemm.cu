// Grouped / dense bf16 GEMM on sm_100a tensor cores.
//
// Persistent, warp-specialised kernel (one CTA per SM):
//   warp 0      TMA producer   (A 128x64 and B BNx64 boxes, 128B swizzle)
//   warp 1      MMA issuer     (one thread, tcgen05.mma kind::f16, M=128, N=BN, K=16)
//   warp 2      TMEM allocator (2 x 256 fp32 accumulator columns)
//   warps 4..7  epilogue       (tcgen05.ld -> fp32 math -> bf16 stores)
// Pipelines: smem ring full/empty (TMA <-> MMA) and a double-buffered TMEM
// accumulator tfull/tempty (MMA <-> epilogue), so the epilogue of tile i
// overlaps the main loop of tile i+1.
//
// The tile list is derived ON DEVICE from the per-group row offsets `seg`
// (expert segments produced by hap_moe_permute), so no host synchronisation is
// needed between the router and the expert GEMMs.  Tiles are ordered m-fastest
// inside each (group, n-block) so concurrently resident CTAs share the weight
// tile through L2.
//
// Models: expert_flops (reference arch.py:165-178) gated-MLP term and the
// projection term of attention_flops (arch.py:157-160).
#include <cstdlib>

#include <cstdio>

#include "common.cuh"

namespace hap {
namespace gemm {

constexpr int BM = 128;  // rows per CTA (a CTA pair covers 2*BM rows)
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle atom row
constexpr int kMaxBN = 256;
constexpr int kMaxSegs = 512;
constexpr int kAccCols = 256;  // TMEM columns per accumulator buffer
constexpr int kThreads = 256;
constexpr int kABytes = BM * BK * 2;  // 16 KB

// Per-CTA pipeline geometry: with a CTA pair each CTA stages only half of the
// B tile, so the same smem holds more stages.
template <int kPair>
struct Geo {
  static constexpr int kBBytes = (kMaxBN / kPair) * BK * 2;  // 32 KB (1 CTA) / 16 KB (pair)
  static constexpr int kStages = kPair == 1 ? 4 : 6;
  static constexpr int kSmemBytes = kStages * (kABytes + kBBytes) + 1024;
};

struct Params {
  int32_t a_rows;
  int32_t K;
  int32_t N;         // B rows per group
  int32_t n_segs;
  int32_t BN;        // n tile (multiple of 16, <= 256)
  int32_t epi;
  int32_t hw;        // swiglu half width (== BN/2 for swiglu)
  int32_t out_cols;  // valid output columns
  const int32_t* seg;
  const int32_t* seg_group;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* resid;
  int64_t ldr;
  // rope epilogue
  const int32_t* positions;
  int32_t head_dim;
  int32_t rope_cols;
  float theta;
  int32_t group_m;  // raster group (m-blocks; < 0: -group_m n-blocks, n fastest)
  uint64_t hint_a, hint_b;  // L2 cache policies of the A / B TMA loads
  int32_t sms;  // SM budget of the launch (persistent grid cap, split-K plan); 0 = all
  int32_t snake;            // serpentine n order across m-groups (HAP_GEMM_SNAKE)
  int32_t noload;           // diagnostics only (HAP_GEMM_NOLOAD): after the first ring fill, stages
                            // complete without TMA loads (MMAs re-read stale smem; results invalid)
  int32_t st32;     // C rows 32-byte aligned: 32-byte stores in the store epilogue
  // split-K (small-M, weight-streaming shapes): each tile's K range is cut in
  // ksplit slices computed by different CTAs; slice ks writes its fp32
  // partial to part[ks][row][col] (row-major over the B rows N) and
  // splitk_reduce_kernel sums the slices in slice order and applies the
  // epilogue — deterministic, no atomics.
  int32_t ksplit;
  float* part;
  // scatter epilogue (EP combine over peer memory): row r of segment s is
  // stored at seg_dst[s] + (r - seg[s] + seg_dst_row0[s]) * ldc, seg_dst[s]
  // being a (possibly peer-mapped) device address; NULL = C
  const int64_t* seg_dst;
  const int32_t* seg_dst_row0;
  // GEMV only (hap_rmsnorm_gemm_qkv_rope): A rows are RMS-normalised with
  // these weights while they are staged in shared memory (same arithmetic as
  // rmsnorm_row_kernel, bit-identical hn); NULL = A is used as is
  const __nv_bfloat16* norm_w;
  float norm_eps;
};

constexpr int kEpiRope = 3;     // internal epilogue id (hap_gemm_qkv_rope)
constexpr int64_t kSplitMax = 16;
constexpr size_t kSplitWorkspaceBytes = (size_t)32 << 20;
constexpr int64_t kSplitDenseMaxRows = 512;  // dense launches up to this many rows may split K
constexpr int64_t kRasterL2Bytes = 48ll << 20;  // A rows of one raster group kept L2-resident across n-blocks

struct TileCoord {
  int32_t g, s, m0, m_end, n_blk;  // weight group, segment, rows [m0, m_end), n block
};

// Map a linear tile index to (segment's weight group, row range, n block).
// tile_start has n_segs+1 prefix entries; m-blocks vary fastest.
template <int TM>
__device__ __forceinline__ TileCoord map_tile(int t, const int32_t* tile_start, const int32_t* seg,
                                              const int32_t* seg_group, int n_segs, int n_blocks, int group_m,
                                              int snake_n = 0) {
  int lo = 0, hi = n_segs - 1;
  while (lo < hi) {  // last g with tile_start[g] <= t
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int g = lo;
  const int local = t - tile_start[g];
  const int rows = seg[g + 1] - seg[g];
  const int m_blocks = (rows + TM - 1) / TM;
  // grouped raster: group_m m-blocks x all n-blocks, m fastest inside a group.
  // group_m is sized so a group's A rows fit the L2 budget: the weight tile of
  // an n-block is then read once per group while the group's A rows stay hot.
  TileCoord c;
  c.g = seg_group[g];
  c.s = g;
  c.m_end = seg[g + 1];
  if (group_m > 0) {
    const int grp = local / (group_m * n_blocks);
    const int g0 = grp * group_m;
    const int gsz = min(group_m, m_blocks - g0);
    const int r = local - grp * group_m * n_blocks;
    c.m0 = seg[g] + (g0 + r % gsz) * TM;
    c.n_blk = r / gsz;
    // serpentine (snake_n): odd m-groups walk the n-blocks backwards, so a group
    // starts on the weight panels the previous group just left in L2
    if (snake_n && (grp & 1)) c.n_blk = n_blocks - 1 - c.n_blk;
  } else {  // n-grouped raster (tuning experiments): -group_m n-blocks x all m-blocks, n fastest
    const int group_n = -group_m;
    const int grp = local / (group_n * m_blocks);
    const int n0 = grp * group_n;
    const int gsz = min(group_n, n_blocks - n0);
    const int r = local - grp * group_n * m_blocks;
    c.n_blk = n0 + r % gsz;
    c.m0 = seg[g] + (r / gsz) * TM;
  }
  return c;
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// kPair == 1: one CTA computes a 128 x BN tile (tcgen05 cta_group::1).
// kPair == 2: a 2-CTA cluster computes a 256 x BN tile with cta_group::2 —
// each CTA stages its 128 A rows and HALF of the B tile (BN/2 rows), the
// leader CTA issues the M=256 MMAs and multicasts the commits, each CTA's
// epilogue drains its own 128 TMEM lanes.  Halving B per SM halves the
// L2->SM operand traffic per FLOP for B.
// kMc == 2 (pair mode only): a cluster of two CTA pairs computes the tiles
// (m, 2j) and (m, 2j+1) of one m-block; the pairs share the A rows, so each
// CTA loads half of its 128-row A slice and multicasts it to the CTA of the
// same pair rank in the other pair (A traffic from L2 halves: 25 % less
// operand traffic per tile).  A stage is reused only after both pairs' MMAs
// consumed it (empty barriers count one commit per pair leader).
template <int kPair, int kMc>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Params p) {
  constexpr int kStages = Geo<kPair>::kStages;
  constexpr int kBBytes = Geo<kPair>::kBBytes;
  constexpr int TM = BM * kPair;  // rows per tile
  constexpr int kCl = kPair * kMc;  // CTAs per cluster
  static_assert(kMc == 1 || kPair == 2, "A multicast is a pair-mode layout");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* smA = smem;
  uint8_t* smB = smem + kStages * kABytes;
  const uint32_t ccta = kCl > 1 ? cluster_ctarank() : 0;
  const uint32_t crank = kPair == 2 ? (ccta & 1) : 0;  // rank inside the CTA pair
  const int pr = kMc == 2 ? (int)(ccta >> 1) : 0;      // pair index inside the cluster
  const bool leader = crank == 0;
  const int tile0 = blockIdx.x / kCl, tile_step = gridDim.x / kCl;

  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ int32_t seg_s[kMaxSegs + 1];
  __shared__ int32_t group_s[kMaxSegs];
  __shared__ int32_t tile_start_s[kMaxSegs + 1];
  __shared__ float inv_freq_s[128];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_segs = p.n_segs;
  const int n_blocks = (p.N + p.BN - 1) / p.BN;
  const int n_sblocks = (n_blocks + kMc - 1) / kMc;  // n-block groups a cluster covers (kMc n-blocks each)
  // PDL: a grouped GEMM's tile list comes from the predecessor (permute's seg),
  // so it waits first; a dense GEMM's does not, and its producer streams the
  // first weight stages before waiting (weights are never written).
  const bool dense = p.seg == nullptr;
  pdl_trigger();
  if (!dense) pdl_wait();

  // ---- setup: segment table, tile prefix, barriers, TMEM
  for (int i = threadIdx.x; i <= n_segs; i += blockDim.x) {
    seg_s[i] = p.seg ? p.seg[i] : (i == 0 ? 0 : p.a_rows);
    if (i < n_segs) group_s[i] = p.seg_group ? p.seg_group[i] : i;
  }
  if (p.epi == kEpiRope) {
    // HF: inv_freq = 1 / theta^(2i/d) in fp32
    for (int i = threadIdx.x; i < p.head_dim / 2; i += blockDim.x)
      inv_freq_s[i] = 1.0f / powf(p.theta, (float)(2 * i) / (float)p.head_dim);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kMc);  // one commit per pair leader reading this stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4 * kPair);  // one arrive per epilogue warp of each CTA
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (kPair == 2) tmem_alloc_pair(&tmem_base_s, 2 * kAccCols);
    else tmem_alloc(&tmem_base_s, 2 * kAccCols);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < n_segs; ++g) {
      tile_start_s[g] = acc;
      const int rows = seg_s[g + 1] - seg_s[g];
      acc += ((rows + TM - 1) / TM) * n_sblocks;
    }
    tile_start_s[n_segs] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (kCl > 1) cluster_sync();  // peer barriers initialised, TMEM allocated in every CTA
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  const int ksplit = p.ksplit;
  const int total_units = tile_start_s[n_segs] * ksplit;
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const int bn_half = p.BN / kPair;
      // the leader's full barrier receives both CTAs' bytes
      const uint32_t tx_bytes = kPair * (kABytes + bn_half * BK * 2);
      int stage = 0;
      uint32_t phase = 0;
      // weight (B) loads of the first stages, issued before the PDL wait
      int npre = 0;
      if (dense && tile0 < total_units) {
        const int t = tile0 / ksplit, ks = tile0 - t * ksplit;
        const TileCoord c = map_tile<TM>(t, tile_start_s, seg_s, group_s, n_segs, n_sblocks, p.group_m, p.snake);
        const int nb = min(c.n_blk * kMc + pr, n_blocks - 1);
        const int b_row = c.g * p.N + nb * p.BN + (int)crank * bn_half;
        const int kb0 = ks * num_kb / ksplit, kb1 = (ks + 1) * num_kb / ksplit;
        npre = min(kStages, kb1 - kb0);
        for (int i = 0; i < npre; ++i) {
          if (kPair == 1) {
            mbar_arrive_expect_tx(&full_bar[i], tx_bytes);
            tma_load_2d(smB + i * kBBytes, &tmB, &full_bar[i], (kb0 + i) * BK, b_row, p.hint_b);
          } else {
            if (leader) mbar_arrive_expect_tx(&full_bar[i], tx_bytes);
            tma_load_2d_pair(smB + i * kBBytes, &tmB, &full_bar[i], (kb0 + i) * BK, b_row, p.hint_b);
          }
        }
      }
      if (dense) pdl_wait();
      for (int u = tile0; u < total_units; u += tile_step) {
        const int t = u / ksplit, ks = u - t * ksplit;
        const TileCoord c = map_tile<TM>(t, tile_start_s, seg_s, group_s, n_segs, n_sblocks, p.group_m, p.snake);
        const int nb = min(c.n_blk * kMc + pr, n_blocks - 1);  // an odd last n-block: pair 1 recomputes it
        // diagnostics (noload == 2): every tile streams the first tile's panels, so
        // the operand traffic stays on L2 and DRAM is idle (results invalid)
        // (noload == 3: only A streams from its real rows; 4: only B)
        const bool fix_b = p.noload == 2 || p.noload == 3, fix_a = p.noload == 2 || p.noload == 4;
        const int b_row = fix_b ? (int)crank * bn_half : c.g * p.N + nb * p.BN + (int)crank * bn_half;
        const int a_row = fix_a ? (int)crank * BM : c.m0 + (int)crank * BM;
        const int kb0 = ks * num_kb / ksplit, kb1 = (ks + 1) * num_kb / ksplit;
        for (int kb = kb0; kb < kb1; ++kb) {
          const bool pre = u == tile0 && kb - kb0 < npre;  // B already in flight
          if (!pre) mbar_wait_spin(&empty_bar[stage], phase ^ 1);
          if (p.noload == 1 && !(u == tile0 && kb - kb0 < kStages)) {  // diagnostics: tensor work without loads
            if (kPair == 1 || leader) mbar_arrive(&full_bar[stage]);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (kPair == 1) {
            if (!pre) mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
            tma_load_2d(smA + stage * kABytes, &tmA, &full_bar[stage], kb * BK, a_row, p.hint_a);
            if (!pre) tma_load_2d(smB + stage * kBBytes, &tmB, &full_bar[stage], kb * BK, b_row, p.hint_b);
          } else {
            if (leader && !pre) mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
            if (kMc == 2)  // this CTA's half of the A slice, to itself and its twin in the other pair
              tma_load_2d_pair_mc(smA + stage * kABytes + pr * (kABytes / 2), &tmA, &full_bar[stage], kb * BK,
                                  a_row + pr * (BM / 2), (uint16_t)((1u << crank) | (1u << (2 + crank))), p.hint_a);
            else
              tma_load_2d_pair(smA + stage * kABytes, &tmA, &full_bar[stage], kb * BK, a_row, p.hint_a);
            if (!pre)
              tma_load_2d_pair(smB + stage * kBBytes, &tmB, &full_bar[stage], kb * BK, b_row, p.hint_b);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0 && leader) {
      const uint32_t idesc = make_idesc_bf16(TM, p.BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = tile0; u < total_units; u += tile_step, ++it) {
        const int ks = u % ksplit;
        const int kb0 = ks * num_kb / ksplit, kb1 = (ks + 1) * num_kb / ksplit;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait_spin(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_spin(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t da = make_sdesc_sw128(smem_u32(smA + stage * kABytes));
          const uint64_t db = make_sdesc_sw128(smem_u32(smB + stage * kBBytes));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 bytes per K=16 step inside the 128B swizzle atom (>>4 => +2)
            if (kPair == 1) umma_bf16_ss(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb != kb0) | (k != 0));
            else umma_bf16_ss_pair(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb != kb0) | (k != 0));
          }
          if (kPair == 1) umma_commit(&empty_bar[stage]);
          else umma_commit_pair_mc(&empty_bar[stage], kMc == 2 ? 0xF : 0x3);  // frees the stage in every CTA that
                                                                             // wrote into this pair's buffers
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (kPair == 1) umma_commit(&tfull_bar[acc]);
        else umma_commit_pair_mc(&tfull_bar[acc], (uint16_t)(0x3u << (2 * pr)));
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    if (dense) pdl_wait();  // reads bias / residual / positions, writes C
    const int q = warp & 3;  // TMEM lane quadrant accessible by this warp
    int it = 0;
    for (int u = tile0; u < total_units; u += tile_step, ++it) {
      const int t = u / ksplit, ks = u - t * ksplit;
      TileCoord c = map_tile<TM>(t, tile_start_s, seg_s, group_s, n_segs, n_sblocks, p.group_m, p.snake);
      const bool dup = c.n_blk * kMc + pr >= n_blocks;  // pair 1's recomputed odd last n-block: no stores
      c.n_blk = min(c.n_blk * kMc + pr, n_blocks - 1);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait_spin(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = c.m0 + (int)crank * BM + q * 32 + lane;
      const bool row_ok = row < c.m_end && !dup;
      const uint32_t t_row = tmem_base + acc * kAccCols + ((uint32_t)(q * 32) << 16);
      __nv_bfloat16* crow =
          p.seg_dst ? reinterpret_cast<__nv_bfloat16*>(p.seg_dst[c.s]) +
                          (int64_t)(row - seg_s[c.s] + p.seg_dst_row0[c.s]) * p.ldc
                    : p.C + (int64_t)row * p.ldc;
      bool do_epi = true;
      if (ksplit > 1 || p.epi == HAP_EPI_F32) {
        // fp32 partials (split-K slice ks) or the raw fp32 accumulator
        // (HAP_EPI_F32: part == C, ksplit == 1, row pitch N).
        // tcgen05.ld is warp-collective: every lane loads, stores are predicated
        do_epi = false;
        float* dst = p.part + ((int64_t)ks * p.a_rows + row) * p.N + c.n_blk * p.BN;
        const int ncols = min(p.BN, p.N - c.n_blk * p.BN);
        for (int j = 0; j < p.BN; j += 32) {
          uint32_t v[32];
          tmem_ld_x32(t_row + j, v);
          tmem_ld_wait();
          if (row_ok) {
            if (p.st32 && (p.N & 7) == 0 && (reinterpret_cast<uintptr_t>(p.part) & 31) == 0) {
#pragma unroll
              for (int i = 0; i < 32; i += 8)
                if (j + i < ncols) {
                  const uint32_t w8[8] = {v[i], v[i + 1], v[i + 2], v[i + 3], v[i + 4], v[i + 5], v[i + 6], v[i + 7]};
                  st_global_v8(dst + j + i, w8);
                }
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                if (j + i < ncols)
                  __stcg(reinterpret_cast<float4*>(dst + j + i),
                         make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                     __uint_as_float(v[i + 3])));
            }
          }
        }
      }
      if (!do_epi) {
      } else if (p.epi == HAP_EPI_SWIGLU) {
        const int hw = p.hw;
        const int col0 = c.n_blk * hw;
        if (p.st32 && (hw & 15) == 0) {
          // 16 output columns per step, one 32-byte store
          for (int j = 0; j < hw; j += 16) {
            uint32_t g[8], g2[8], u[8], u2[8];
            tmem_ld_x8(t_row + j, g);
            tmem_ld_x8(t_row + j + 8, g2);
            tmem_ld_x8(t_row + hw + j, u);
            tmem_ld_x8(t_row + hw + j + 8, u2);
            tmem_ld_wait();
            if (row_ok && col0 + j < p.out_cols) {
              uint32_t o[8];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                o[i] = pack_bf16x2(silu(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]),
                                   silu(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]));
                o[4 + i] = pack_bf16x2(silu(__uint_as_float(g2[2 * i])) * __uint_as_float(u2[2 * i]),
                                       silu(__uint_as_float(g2[2 * i + 1])) * __uint_as_float(u2[2 * i + 1]));
              }
              if (col0 + j + 16 <= p.out_cols) {
                st_global_v8(crow + col0 + j, o);
              } else {
                *reinterpret_cast<uint4*>(crow + col0 + j) = make_uint4(o[0], o[1], o[2], o[3]);
                if (col0 + j + 8 < p.out_cols)
                  *reinterpret_cast<uint4*>(crow + col0 + j + 8) = make_uint4(o[4], o[5], o[6], o[7]);
              }
            }
          }
        } else {
          for (int j = 0; j < hw; j += 8) {
            uint32_t g[8], u[8];
            tmem_ld_x8(t_row + j, g);
            tmem_ld_x8(t_row + hw + j, u);
            tmem_ld_wait();
            if (row_ok && col0 + j < p.out_cols) {
              uint32_t o[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float a0 = silu(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
                const float a1 = silu(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
                o[i] = pack_bf16x2(a0, a1);
              }
              *reinterpret_cast<uint4*>(crow + col0 + j) = make_uint4(o[0], o[1], o[2], o[3]);
            }
          }
        }
      } else if (p.epi == kEpiRope) {
        // QKV projection with fused rotary embedding on the q/k head columns:
        // tile = BN/d whole heads; pairs (i, i + d/2) of a head are rotated by
        // pos*inv_freq[i] (fp32), bias added first, one bf16 rounding.
        const int d = p.head_dim, half = d >> 1;
        const int col0 = c.n_blk * p.BN;
        const float pos = row_ok ? (float)p.positions[row] : 0.f;
        for (int hb = 0; hb < p.BN; hb += d) {
          const int hcol = col0 + hb;
          const bool rot = hcol < p.rope_cols;
          // 8 rotation pairs per sub-step; with 32-byte stores two sub-steps
          // (16 columns of each half) leave together
          const bool wide = p.st32 && (half % 16) == 0;
          for (int i = 0; i < half; i += (wide ? 16 : 8)) {
            uint32_t o1w[8], o2w[8];
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              if (sub == 1 && !wide) break;
              const int ii = i + sub * 8;
              uint32_t a[8], b[8];
              tmem_ld_x8(t_row + hb + ii, a);
              tmem_ld_x8(t_row + hb + half + ii, b);
              tmem_ld_wait();
              if (!row_ok || hcol >= p.out_cols) continue;
              float x1[8], x2[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                x1[k] = __uint_as_float(a[k]);
                x2[k] = __uint_as_float(b[k]);
              }
              if (p.bias) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  x1[k] += __bfloat162float(p.bias[hcol + ii + k]);
                  x2[k] += __bfloat162float(p.bias[hcol + half + ii + k]);
                }
              }
              if (rot) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  float sn, cs;
                  rope_sincos(pos * inv_freq_s[ii + k], &sn, &cs);
                  const float y1 = x1[k] * cs - x2[k] * sn;
                  const float y2 = x2[k] * cs + x1[k] * sn;
                  x1[k] = y1;
                  x2[k] = y2;
                }
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                o1w[sub * 4 + k] = pack_bf16x2(x1[2 * k], x1[2 * k + 1]);
                o2w[sub * 4 + k] = pack_bf16x2(x2[2 * k], x2[2 * k + 1]);
              }
            }
            if (!row_ok || hcol >= p.out_cols) continue;
            if (wide) {
              st_global_v8(crow + hcol + i, o1w);
              st_global_v8(crow + hcol + half + i, o2w);
            } else {
              *reinterpret_cast<uint4*>(crow + hcol + i) = make_uint4(o1w[0], o1w[1], o1w[2], o1w[3]);
              *reinterpret_cast<uint4*>(crow + hcol + half + i) = make_uint4(o2w[0], o2w[1], o2w[2], o2w[3]);
            }
          }
        }
      } else {
        const int col0 = c.n_blk * p.BN;
        for (int j = 0; j < p.BN; j += 32) {
          uint32_t v[32];
          tmem_ld_x32(t_row + j, v);
          tmem_ld_wait();
          if (row_ok) {
            uint32_t o32[8];  // two 8-column groups gathered for one 32-byte store
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int col = col0 + j + s * 8;
              const bool pair32 = p.st32 && ((s & 1) ? col - 8 : col + 8) < p.out_cols;
              if (col < p.out_cols) {
                float f[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[s * 8 + i]);
                if (p.bias) {
                  const uint4 b = *reinterpret_cast<const uint4*>(p.bias + col);
                  const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const float2 bb = unpack_bf16x2(bw[i]);
                    f[2 * i] += bb.x;
                    f[2 * i + 1] += bb.y;
                  }
                }
                if (p.resid) {
                  const uint4 r = *reinterpret_cast<const uint4*>(p.resid + (int64_t)row * p.ldr + col);
                  const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const float2 rr = unpack_bf16x2(rw[i]);
                    f[2 * i] += rr.x;
                    f[2 * i + 1] += rr.y;
                  }
                }
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) o[i] = pack_bf16x2(f[2 * i], f[2 * i + 1]);
                if (pair32) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) o32[(s & 1) * 4 + i] = o[i];
                  if (s & 1) st_global_v8(crow + col - 8, o32);
                } else {
                  *reinterpret_cast<uint4*>(crow + col) = make_uint4(o[0], o[1], o[2], o[3]);
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // accumulator drained by this warp -> the leader's MMA may reuse it
        if (kPair == 1) mbar_arrive(&tempty_bar[acc]);
        else mbar_arrive_cluster(&tempty_bar[acc], ccta & ~1u);  // this pair's leader
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (kCl > 1) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if (kPair == 2) tmem_dealloc_pair(tmem_base, 2 * kAccCols);
    else tmem_dealloc(tmem_base, 2 * kAccCols);
  }
}

// Pick the n tile: the largest multiple of 16 <= 256 that divides N (so no
// weight tile straddles two groups' rows wastefully); fall back to 256 with
// column masking.
static int pick_bn(int64_t N) {
  for (int bn = 256; bn >= 64; bn -= 16)
    if (N % bn == 0) return bn;
  return N < 256 ? (int)((N + 15) / 16 * 16) : 256;
}

// ---- split-K reduction + epilogue (phase 2) --------------------------------
// One thread per 8 outputs of a row: sums the fp32 slice partials in slice
// order, then the same epilogue math as the TMEM path (bias, residual, SwiGLU,
// RoPE with inv_freq = 1/theta^(2i/d)), one bf16 rounding.
__device__ __forceinline__ void sum_slices8(const float* part, int64_t slice, int ks, int64_t off, float (&f)[8]) {
  // slices are loaded 8 at a time with every load in flight before the first
  // add (ks/8 memory round trips instead of ks); the sum order is slice order
  constexpr int kB = 8;
  for (int s0 = 0; s0 < ks; s0 += kB) {
    float4 a[kB], b[kB];
#pragma unroll
    for (int s = 0; s < kB; ++s) {
      if (s0 + s < ks) {
        a[s] = __ldcg(reinterpret_cast<const float4*>(part + (s0 + s) * slice + off));
        b[s] = __ldcg(reinterpret_cast<const float4*>(part + (s0 + s) * slice + off + 4));
      }
    }
#pragma unroll
    for (int s = 0; s < kB; ++s) {
      if (s0 + s >= ks) break;
      if (s0 + s == 0) {
        f[0] = a[0].x; f[1] = a[0].y; f[2] = a[0].z; f[3] = a[0].w;
        f[4] = b[0].x; f[5] = b[0].y; f[6] = b[0].z; f[7] = b[0].w;
      } else {
        f[0] += a[s].x; f[1] += a[s].y; f[2] += a[s].z; f[3] += a[s].w;
        f[4] += b[s].x; f[5] += b[s].y; f[6] += b[s].z; f[7] += b[s].w;
      }
    }
  }
}

__global__ void __launch_bounds__(256) splitk_reduce_kernel(Params p) {
  pdl_trigger();
  pdl_wait();
  const int N = p.N;
  const int items = p.epi == HAP_EPI_SWIGLU ? N / 16 : (p.epi == kEpiRope ? N / 16 : N / 8);
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(idx / items), it = (int)(idx % items);
  if (row >= p.a_rows) return;
  if (p.seg && (row < p.seg[0] || row >= p.seg[p.n_segs])) return;
  const int64_t slice = (int64_t)p.a_rows * N;
  const int64_t rbase = (int64_t)row * N;
  __nv_bfloat16* crow = p.C + (int64_t)row * p.ldc;
  if (p.epi == HAP_EPI_SWIGLU) {
    const int hw = p.hw, o = it * 8, j = o / hw, i0 = o % hw;
    float g[8], u[8];
    sum_slices8(p.part, slice, p.ksplit, rbase + j * 2 * hw + i0, g);
    sum_slices8(p.part, slice, p.ksplit, rbase + j * 2 * hw + hw + i0, u);
    uint32_t out[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = pack_bf16x2(silu(g[2 * i]) * u[2 * i], silu(g[2 * i + 1]) * u[2 * i + 1]);
    *reinterpret_cast<uint4*>(crow + o) = make_uint4(out[0], out[1], out[2], out[3]);
  } else if (p.epi == kEpiRope) {
    const int d = p.head_dim, half = d >> 1, per_head = half / 8;
    const int hcol = (it / per_head) * d, i0 = (it % per_head) * 8;
    float x1[8], x2[8];
    sum_slices8(p.part, slice, p.ksplit, rbase + hcol + i0, x1);
    sum_slices8(p.part, slice, p.ksplit, rbase + hcol + half + i0, x2);
    if (p.bias) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        x1[k] += __bfloat162float(p.bias[hcol + i0 + k]);
        x2[k] += __bfloat162float(p.bias[hcol + half + i0 + k]);
      }
    }
    if (hcol < p.rope_cols) {
      const float pos = (float)p.positions[row];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float inv_freq = 1.0f / powf(p.theta, (float)(2 * (i0 + k)) / (float)d);
        float sn, cs;
        rope_sincos(pos * inv_freq, &sn, &cs);
        const float y1 = x1[k] * cs - x2[k] * sn;
        const float y2 = x2[k] * cs + x1[k] * sn;
        x1[k] = y1;
        x2[k] = y2;
      }
    }
    uint32_t o1[4], o2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o1[k] = pack_bf16x2(x1[2 * k], x1[2 * k + 1]);
      o2[k] = pack_bf16x2(x2[2 * k], x2[2 * k + 1]);
    }
    *reinterpret_cast<uint4*>(crow + hcol + i0) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
    *reinterpret_cast<uint4*>(crow + hcol + half + i0) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
  } else {
    const int col = it * 8;
    float f[8];
    sum_slices8(p.part, slice, p.ksplit, rbase + col, f);
    if (p.bias) {
      const uint4 b = *reinterpret_cast<const uint4*>(p.bias + col);
      const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 bb = unpack_bf16x2(bw[i]);
        f[2 * i] += bb.x;
        f[2 * i + 1] += bb.y;
      }
    }
    if (p.resid) {
      const uint4 r = *reinterpret_cast<const uint4*>(p.resid + (int64_t)row * p.ldr + col);
      const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 rr = unpack_bf16x2(rw[i]);
        f[2 * i] += rr.x;
        f[2 * i + 1] += rr.y;
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = pack_bf16x2(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(crow + col) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Choose (BN, ksplit) for a single-CTA launch whose tiles cannot cover the
// SMs: the smallest split reaching ~85% of the SMs (fewest partial bytes),
// preferring the larger tile; partials must fit the workspace.
static void plan_split(Params& p, int64_t a_rows, int64_t K, int64_t N, int64_t n_segs, size_t ws_bytes) {
  p.ksplit = 1;
  const int64_t nsm = p.sms > 0 ? p.sms : kNumSMs;
  auto tiles = [&](int64_t bn) { return ((a_rows + BM - 1) / BM + (n_segs - 1)) * ((N + bn - 1) / bn); };
  if (N % 8) return;
  const int64_t num_kb = (K + BK - 1) / BK;
  if (2 * tiles(p.BN) > nsm) {
    // Many tiles, but a badly quantised last wave (e.g. 160 tiles = 1.08 waves
    // on 148 SMs: the weight stream takes two rounds).  A grouped launch has at
    // most min(rows, segments) non-empty segments, one m-block each here
    // (a_rows <= BM), which bounds its real tile count without a host sync.
    const int64_t n_blocks = (N + p.BN - 1) / p.BN;
    const int64_t t = p.seg == nullptr ? ((a_rows + BM - 1) / BM) * n_blocks
                                       : (a_rows < n_segs ? a_rows : n_segs) * n_blocks;
    auto rounds = [&](int64_t ks) { return (double)((t * ks + nsm - 1) / nsm) / (double)ks; };
    int64_t best = 1;
    for (int64_t ks = 2; ks <= 8 && ks <= num_kb / 4; ++ks)
      if ((size_t)ks * a_rows * N * sizeof(float) <= ws_bytes && rounds(ks) < rounds(best)) best = ks;
    if (rounds(best) <= 0.85 * rounds(1)) p.ksplit = (int32_t)best;
    return;
  }
  int64_t cands[3] = {p.BN, 0, 0};
  int nc = 1;
  if (p.epi == HAP_EPI_STORE) {
    for (int64_t bn : {(int64_t)128, (int64_t)64})
      if (bn < p.BN && N % bn == 0) cands[nc++] = bn;
  } else if (p.epi == kEpiRope && p.head_dim < p.BN) {
    cands[nc++] = p.head_dim;
  }
  int64_t best_bn = p.BN, best_ks = 1, best_units = tiles(p.BN);
  bool best_ok = false;
  for (int c = 0; c < nc; ++c) {
    const int64_t t = tiles(cands[c]);
    int64_t ks = nsm / t;
    if (ks > num_kb / 4) ks = num_kb / 4;  // >= 4 k-blocks (256 K) per slice
    if (ks > kSplitMax) ks = kSplitMax;
    while (ks > 1 && (size_t)ks * a_rows * N * sizeof(float) > ws_bytes) --ks;
    if (ks < 1) ks = 1;
    const int64_t units = t * ks;
    const bool ok = units * 100 >= nsm * 85;
    if ((ok && (!best_ok || ks < best_ks)) || (!ok && !best_ok && units > best_units)) {
      best_bn = cands[c];
      best_ks = ks;
      best_units = units;
      best_ok = ok;
    }
  }
  if (best_ks > 1) {
    p.BN = (int32_t)best_bn;
    p.ksplit = (int32_t)best_ks;
  }
}

template <int kPair, int kMc = 1>
static int launch_impl(Params& p, const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                       int64_t n_groups, int64_t N, int64_t n_segs, void* stream) {
  constexpr int TM = BM * kPair;
  constexpr int kCl = kPair * kMc;
  CUtensorMap tmA, tmB;
  if (!encode_tmap_2d_bf16(&tmA, A, (uint64_t)K, (uint64_t)a_rows, (uint64_t)lda * 2, BK, BM / kMc, true))
    return HAP_ERR_DRIVER;
  if (!encode_tmap_2d_bf16(&tmB, B, (uint64_t)K, (uint64_t)(n_groups * N), (uint64_t)K * 2, BK, p.BN / kPair,
                           true))
    return HAP_ERR_DRIVER;
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)grouped_gemm_kernel<kPair, kMc>, Geo<kPair>::kSmemBytes) != 0)
      return HAP_ERR_LAUNCH;
    configured = 1;
  }
  // Upper bound on tiles without reading seg on the host.
  const int64_t n_blocks = (N + p.BN - 1) / p.BN;
  static const int64_t l2_budget = [] {
    const char* e = getenv("HAP_GEMM_RASTER_MB");  // tuning experiments only
    return e ? (int64_t)atoi(e) << 20 : kRasterL2Bytes;
  }();
  static const bool st32_ok = [] {
    const char* e = getenv("HAP_GEMM_ST32");  // A/B experiments only
    return !(e && e[0] == '0');
  }();
  p.st32 = (st32_ok && p.seg_dst == nullptr && p.C != nullptr &&
            ((reinterpret_cast<uintptr_t>(p.C) | (uintptr_t)(p.ldc * 2)) & 31) == 0) ? 1 : 0;
  // tuning experiments only: HAP_GEMM_HINT=<A><B> with N(ormal) / F(irst) / L(ast)
  // L2 eviction priorities, HAP_GEMM_RASTER_N=1 for the n-grouped raster
  static const uint64_t hints[2] = {[] {
    const char* e = getenv("HAP_GEMM_HINT");
    return e && e[0] == 'F' ? kEvictFirst : (e && e[0] == 'L' ? kEvictLast : kEvictNormal);
  }(), [] {
    const char* e = getenv("HAP_GEMM_HINT");
    return e && e[0] && e[1] == 'F' ? kEvictFirst : (e && e[0] && e[1] == 'L' ? kEvictLast : kEvictNormal);
  }()};
  static const bool raster_n = [] {
    const char* e = getenv("HAP_GEMM_RASTER_N");
    return e && e[0] == '1';
  }();
  p.hint_a = hints[0];
  p.hint_b = hints[1];
  static const int noload = [] {
    const char* e = getenv("HAP_GEMM_NOLOAD");  // diagnostics only: results are invalid
    return e ? atoi(e) : 0;
  }();
  p.noload = noload;
  static const int snake = [] {
    // A/B switch, default on: the down GEMM at the power cap 1290 -> 1315 TF/s,
    // DRAM reads 5.0-6.4 -> 4.6-5.4 GB (tile order only: results unchanged)
    const char* e = getenv("HAP_GEMM_SNAKE");
    return e ? atoi(e) : 1;
  }();
  p.snake = snake;
  int64_t gm = l2_budget / (K * 2 * (raster_n ? (int64_t)p.BN : (int64_t)TM));
  p.group_m = (int32_t)(gm < 1 ? 1 : (gm > 1024 ? 1024 : gm));
  if (raster_n) p.group_m = -p.group_m;
  const int64_t max_tiles = ((a_rows + TM - 1) / TM + (n_segs - 1)) * ((n_blocks + kMc - 1) / kMc);
  // persistent grid = the clusters that can be co-resident (4-CTA clusters do
  // not tile every GPC: 33 of them fit on 148 SMs, not 37)
  static const int64_t max_units = [] {
    if (kCl <= 2) return (int64_t)(kNumSMs / kCl);
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(kNumSMs);
    q.blockDim = dim3(kThreads);
    q.dynamicSmemBytes = Geo<kPair>::kSmemBytes;
    cudaLaunchAttribute a{};
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = kCl;
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = 1;
    q.attrs = &a;
    q.numAttrs = 1;
    int n_cl = 0;
    if (cudaOccupancyMaxActiveClusters(&n_cl, (void*)grouped_gemm_kernel<kPair, kMc>, &q) != cudaSuccess || n_cl < 1)
      n_cl = kNumSMs / kCl;
    return (int64_t)n_cl;
  }();
  const int64_t units = max_tiles * p.ksplit;
  const int64_t cap_units = p.sms > 0 && p.sms / kCl < max_units ? (p.sms / kCl > 0 ? p.sms / kCl : 1) : max_units;
  const int grid = (int)((units < cap_units ? units : cap_units) * kCl);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Geo<kPair>::kSmemBytes;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_for(a_rows) || (pdl_mode() == 2 && p.seg == nullptr)) ? 2 : 1;
  static const bool debug = getenv("HAP_GEMM_DEBUG") != nullptr;
  if (debug) {
    int n_cl = -1;
    cudaOccupancyMaxActiveClusters(&n_cl, (void*)grouped_gemm_kernel<kPair, kMc>, &cfg);
    fprintf(stderr, "[hap gemm] cluster %d: max active clusters %d, grid %d CTAs\n", kCl, n_cl, grid);
  }
  if (cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<kPair, kMc>, tmA, tmB, p) != cudaSuccess) return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

// A multicast across two CTA pairs (kMc = 2): HAP_GEMM_MC=1 (A/B switch)
static bool a_multicast() {
  static const bool on = [] {
    const char* e = getenv("HAP_GEMM_MC");
    return e && e[0] == '1' && !getenv("HAP_GEMM_NOLOAD");  // the load diagnostics are 1-pair layouts
  }();
  return on;
}

static int pair_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("HAP_GEMM_CTA_PAIR");  // A/B switch for profiling; default on
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode;
}


// ---- small-M weight streaming (decode) -------------------------------------
// a_rows <= 8: every weight row is read once by one warp that dots it with all
// the (<= 8) activation rows held in shared memory, 16-byte loads, 4 chunks in
// flight per lane, fp32 accumulation per lane in k order then a fixed xor-
// shuffle tree (deterministic).  A warp item is a PAIR of weight rows so every
// epilogue closes inside the item: two output columns (store / bias /
// residual), the gate and up rows of one SwiGLU column, or the columns i and
// i + d/2 of one rotary head.  Grouped launches: items run over (segment,
// column pair), rows of segment s dotted with weight group seg_group[s].
// Replaces the 128-row tensor-core tile + split-K + reduce launches whose
// fill / drain dominate decode projections (Qwen2-57B B=1 QKV: 15.5 + 6.8 us).
constexpr int kGvThreads = 256;
constexpr int kGvMaxRows = 8;
constexpr int kGvU = 4;  // 16-byte chunks in flight per lane and weight row

__device__ __forceinline__ void gv_dot8(const uint4 w, const uint4 x, float& acc) {
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  const uint32_t xx[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 a = unpack_bf16x2(ww[q]);
    const float2 b = unpack_bf16x2(xx[q]);
    acc = fmaf(a.x, b.x, acc);
    acc = fmaf(a.y, b.y, acc);
  }
}

// Stage the (<= 8) activation rows of a GEMV launch in shared memory, RMS-
// normalised on the way when p.norm_w is set: the first 128 threads
// normalise the rows one after the other with exactly rmsnorm_row_kernel's
// order (thread t: vectors t, t+128, ...; fma x then y per bf16 pair; xor-
// shuffle tree; (w0 + w1) + (w2 + w3)) — bit-identical to hap_rmsnorm.
// Called by every thread of the CTA (contains __syncthreads).
__device__ __forceinline__ void gv_stage_rows(uint4* xs, const __nv_bfloat16* __restrict__ A, int64_t lda,
                                              const Params& p, int kv) {
  if (p.norm_w) {
    __shared__ float red[4];
    const int t = threadIdx.x, lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint4* nw = reinterpret_cast<const uint4*>(p.norm_w);
    for (int r = 0; r < p.a_rows; ++r) {  // one row at a time on the first 128 threads
      const bool mine = t < 128;
      const uint4* xr = reinterpret_cast<const uint4*>(A + (int64_t)r * lda);
      float ss = 0.f;
      if (mine) {
        for (int c = t; c < kv; c += 128) {
          const uint4 v = __ldg(xr + c);
          const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(u[j]);
            ss = fmaf(f.x, f.x, ss);
            ss = fmaf(f.y, f.y, ss);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (mine && lane == 0) red[wq] = ss;
      __syncthreads();
      if (mine) {
        const float tot = (red[0] + red[1]) + (red[2] + red[3]);
        const float inv = rsqrtf(tot / (float)(kv * 8) + p.norm_eps);
        for (int c = t; c < kv; c += 128) {
          const uint4 v = __ldg(xr + c), wv = __ldg(nw + c);
          const uint32_t u[4] = {v.x, v.y, v.z, v.w};
          const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
          uint32_t o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(u[j]);
            const float2 g = unpack_bf16x2(ww[j]);
            o[j] = pack_bf16x2(f.x * inv * g.x, f.y * inv * g.y);
          }
          xs[r * kv + c] = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      __syncthreads();
    }
  } else {
    for (int i = threadIdx.x; i < p.a_rows * kv; i += blockDim.x) {
      const int r = i / kv, c = i - r * kv;
      xs[i] = *reinterpret_cast<const uint4*>(A + (int64_t)r * lda + (int64_t)c * 8);
    }
    __syncthreads();
  }
}

// The two weight rows of GEMV item (column pair) c2: the two output columns,
// the gate and up rows of one SwiGLU column, or columns i and i + d/2 of a head.
__device__ __forceinline__ void gv_rows(const Params& p, int c2, int& na, int& nb) {
  if (p.epi == HAP_EPI_SWIGLU) {
    na = (c2 / p.hw) * 2 * p.hw + c2 % p.hw;
    nb = na + p.hw;
  } else if (p.epi == kEpiRope) {
    const int d = p.head_dim, half = d >> 1;
    na = (c2 / half) * d + c2 % half;
    nb = na + half;
  } else {
    na = 2 * c2;
    nb = na + 1;
  }
}

// Epilogue of one (row, column pair): SwiGLU / bias / RoPE / residual, bf16 out.
__device__ __forceinline__ void gv_store(const Params& p, int row, int c2, int na, int nb, float x1, float x2) {
  __nv_bfloat16* crow = p.C + (int64_t)row * p.ldc;
  if (p.epi == HAP_EPI_SWIGLU) {
    crow[c2] = __float2bfloat16_rn(silu(x1) * x2);
    return;
  }
  if (p.bias) {
    x1 += __bfloat162float(p.bias[na]);
    x2 += __bfloat162float(p.bias[nb]);
  }
  if (p.epi == kEpiRope) {
    const int d = p.head_dim, half = d >> 1;
    if (na < p.rope_cols) {
      const int i = c2 % half;
      const float inv_freq = 1.0f / powf(p.theta, (float)(2 * i) / (float)d);
      float sn, cs;
      rope_sincos((float)p.positions[row] * inv_freq, &sn, &cs);
      const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
      x1 = y1;
      x2 = y2;
    }
    crow[na] = __float2bfloat16_rn(x1);
    crow[nb] = __float2bfloat16_rn(x2);
    return;
  }
  if (p.resid) {
    x1 += __bfloat162float(p.resid[(int64_t)row * p.ldr + na]);
    x2 += __bfloat162float(p.resid[(int64_t)row * p.ldr + nb]);
  }
  *reinterpret_cast<uint32_t*>(crow + na) = pack_bf16x2(x1, x2);
}

// kR: the launch's row bound (2 for the default 1-2-row decode launches: 4
// accumulators instead of 16 keep the kernel under ~96 registers so 3072
// warps of a 50 MB QKV stream are resident in one round; same arithmetic per
// row for every kR, so the results do not depend on it)
template <int kR>
__global__ void __launch_bounds__(kGvThreads, kR <= 2 ? 3 : 1) gemv_kernel(const __nv_bfloat16* __restrict__ A, int64_t lda,
                                                          const __nv_bfloat16* __restrict__ B, Params p) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ uint4 xs[];  // [a_rows][K/8]
  const int kv = p.K / 8;
  gv_stage_rows(xs, A, lda, p, kv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pairs = p.N / 2;  // column pairs per segment
  const int n_items = p.n_segs * n_pairs;
  for (int item = blockIdx.x * (kGvThreads / 32) + warp; item < n_items; item += gridDim.x * (kGvThreads / 32)) {
    const int s = item / n_pairs, c2 = item - s * n_pairs;
    const int r0 = p.seg ? p.seg[s] : 0, r1 = p.seg ? p.seg[s + 1] : p.a_rows;
    if (r1 <= r0) continue;
    const int g = p.seg_group ? p.seg_group[s] : s;
    int na, nb;  // the two weight rows of this item
    gv_rows(p, c2, na, nb);
    const uint4* wa = reinterpret_cast<const uint4*>(B + ((int64_t)g * p.N + na) * p.K);
    const uint4* wb = reinterpret_cast<const uint4*>(B + ((int64_t)g * p.N + nb) * p.K);
    const int nr = r1 - r0;
    float acc_a[kR], acc_b[kR];
#pragma unroll
    for (int m = 0; m < kR; ++m) acc_a[m] = acc_b[m] = 0.f;
    // software-pipelined: the next group of chunks is in flight while this one
    // is consumed (two groups = 8 KB per warp outstanding)
    uint4 va[kGvU], vb[kGvU];
#pragma unroll
    for (int u = 0; u < kGvU; ++u) {
      const int c = lane + 32 * u;
      va[u] = c < kv ? __ldg(wa + c) : make_uint4(0, 0, 0, 0);
      vb[u] = c < kv ? __ldg(wb + c) : make_uint4(0, 0, 0, 0);
    }
    for (int c0 = lane; c0 < kv; c0 += 32 * kGvU) {
      uint4 na_[kGvU], nb_[kGvU];
#pragma unroll
      for (int u = 0; u < kGvU; ++u) {
        const int c = c0 + 32 * (kGvU + u);
        na_[u] = c < kv ? __ldg(wa + c) : make_uint4(0, 0, 0, 0);
        nb_[u] = c < kv ? __ldg(wb + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kGvU; ++u) {
        const int c = c0 + 32 * u;
        if (c >= kv) break;
#pragma unroll
        for (int m = 0; m < kR; ++m) {
          if (m < nr) {
            const uint4 x = xs[(r0 + m) * kv + c];
            gv_dot8(va[u], x, acc_a[m]);
            gv_dot8(vb[u], x, acc_b[m]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kGvU; ++u) {
        va[u] = na_[u];
        vb[u] = nb_[u];
      }
    }
#pragma unroll
    for (int m = 0; m < kR; ++m) {
      if (m < nr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc_a[m] += __shfl_xor_sync(0xffffffffu, acc_a[m], o);
          acc_b[m] += __shfl_xor_sync(0xffffffffu, acc_b[m], o);
        }
      }
    }
    // epilogue: lane m writes row r0 + m
#pragma unroll
    for (int m = 0; m < kR; ++m) {
      if (m != lane || m >= nr) continue;
      gv_store(p, r0 + m, c2, na, nb, acc_a[m], acc_b[m]);
    }
  }
}

// HAP_GEMV: 0 = tensor-core tiles for every M; 1 (default) = GEMV for launches
// of <= 2 activation rows streaming <= 64 MB of weights (decode QKV / O at
// batch 1-2); 2 = GEMV for every eligible launch of <= 8 rows (experiments).
// Per launch from HBM the GEMV wins at 1-2 rows on those streams and loses on
// the long expert streams and at 4-8 rows; in the graph-replayed decode block
// it measured Qwen2-57B B=1 226 -> 215 us, Mixtral-8x7B B=1 223 -> 205 us once
// the shared expert kept to half the SMs (profiles/r02_gemv_ab.txt)
constexpr int64_t kGvAutoRows = 2;
static int gemv_mode() {
  static const int mode = [] {
    const char* e = getenv("HAP_GEMV");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

static int launch_gemv(Params& p, const void* A, int64_t lda, const void* B, void* stream) {
  const int smem = p.a_rows * p.K * 2;
  static int configured = 0;
  if (!configured) {
    if (configure_smem((const void*)gemv_kernel<2>, 200 * 1024)) return HAP_ERR_LAUNCH;
    if (configure_smem((const void*)gemv_kernel<kGvMaxRows>, 200 * 1024)) return HAP_ERR_LAUNCH;
    configured = 1;
  }
  auto kern = p.a_rows <= 2 ? gemv_kernel<2> : gemv_kernel<kGvMaxRows>;
  const int64_t items = (int64_t)p.n_segs * (p.N / 2);
  int64_t ctas = (items + (kGvThreads / 32) - 1) / (kGvThreads / 32);
  const int per_sm = smem > 0 ? (int)((220 * 1024) / (smem + 1024)) : 8;
  const int64_t cap = (int64_t)kNumSMs * (per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm));
  if (ctas > cap) ctas = cap;
  if (hap::launch_kr(p.a_rows, kern, dim3((unsigned)ctas), dim3(kGvThreads), smem, reinterpret_cast<cudaStream_t>(stream),
                    reinterpret_cast<const __nv_bfloat16*>(A), lda, reinterpret_cast<const __nv_bfloat16*>(B),
                    p) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

static int launch(Params& p, const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                  int64_t n_groups, int64_t N, int64_t n_segs, void* ws, size_t ws_bytes, void* stream) {
  // CTA pairs need B split in two whole 8-row swizzle groups, and only pay off
  // when segments fill 256-row tiles (prefill); weight-streaming decode shapes
  // (a few rows per expert) keep 128-row single-CTA tiles.
  p.ksplit = 1;
  // decode-size launches (<= 8 activation rows in all), HAP_GEMV=1|2: one warp
  // per weight-row pair, no tensor-core tiles (see gemv_kernel / gemv_mode)
  if (gemv_mode() > 0 && a_rows <= kGvMaxRows && p.seg_dst == nullptr && p.epi != HAP_EPI_F32 && p.N % 2 == 0 &&
      a_rows * K * 2 <= 192 * 1024 && (p.epi != HAP_EPI_SWIGLU || p.hw > 0) &&
      (gemv_mode() == 2 || (a_rows <= kGvAutoRows && n_groups * N * K * 2 <= (int64_t)64 << 20)))
    return launch_gemv(p, A, lda, B, stream);
  // Dense launches of a few hundred rows (decode at large batch: QKV / O at
  // T = 512 are 36 / 28 pair tiles on 148 SMs) split K over 1-CTA tiles when
  // that fills the GPU.  Opt-in (HAP_GEMM_SPLIT_DENSE=1): the K split changes
  // the fp32 summation order, so a 256-row prefill chunk would no longer be
  // bit-identical to the same rows inside a larger launch
  // (test_forward_host_streams_chunks_identically), for a gain within a few %
  static const bool split_dense = [] {
    const char* e = getenv("HAP_GEMM_SPLIT_DENSE");
    return e && e[0] == '1';
  }();
  bool dense_split = false;
  if (split_dense && ws && ws_bytes >= 16 && p.seg == nullptr && a_rows > BM && a_rows <= kSplitDenseMaxRows &&
      p.epi != HAP_EPI_F32) {
    Params q = p;
    plan_split(q, a_rows, K, N, n_segs, ws_bytes);
    if (q.ksplit > 1) {
      p = q;
      dense_split = true;
    }
  }
  if (!dense_split && pair_mode() && (p.BN / 2) % 8 == 0 && a_rows >= 256 * n_segs) {
    if (a_multicast() && (N + p.BN - 1) / p.BN >= 2)
      return launch_impl<2, 2>(p, A, a_rows, lda, K, B, n_groups, N, n_segs, stream);
    return launch_impl<2>(p, A, a_rows, lda, K, B, n_groups, N, n_segs, stream);
  }
  // Small-M weight streaming (decode projections, TP-sharded shapes): split K
  // over more CTAs when a workspace is supplied, then reduce + epilogue.
  // Only single-m-block launches split; the slice plan depends on (N, K, M) only
  // through the tile bound and the workspace fit, and repeats bit for bit.
  if (dense_split) {
    p.part = reinterpret_cast<float*>(ws);
  } else if (ws && ws_bytes >= 16 && a_rows <= BM) {
    plan_split(p, a_rows, K, N, n_segs, ws_bytes);
    p.part = reinterpret_cast<float*>(ws);
  }
  const int st = launch_impl<1>(p, A, a_rows, lda, K, B, n_groups, N, n_segs, stream);
  if (st != HAP_OK || p.ksplit == 1) return st;
  const int items = p.epi == HAP_EPI_STORE ? (int)(N / 8) : (int)(N / 16);
  const int64_t threads = a_rows * items;
  { if (hap::launch_kr(a_rows, splitk_reduce_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0,
               reinterpret_cast<cudaStream_t>(stream), p) != cudaSuccess)
    return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

}  // namespace gemm
}  // namespace hap

using namespace hap;

extern "C" int64_t hap_swiglu_half_width(int64_t inter_dim) {
  if (inter_dim <= 0 || inter_dim % 8) return -1;
  for (int64_t hw = 128; hw >= 8; hw -= 8)
    if (inter_dim % hw == 0) return hw;
  return -1;
}

extern "C" size_t hap_gemm_splitk_workspace_bytes(void) {
  return hap::gemm::kSplitWorkspaceBytes;
}

extern "C" int hap_grouped_gemm_bf16_ex(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                                        int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                                        const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                                        int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                                        void* workspace, size_t ws_bytes, void* stream) {
  return hap_grouped_gemm_bf16_sms(A, a_rows, lda, K, B, n_groups, N, seg, n_segs, seg_group, C, ldc, epilogue,
                                   swiglu_half, bias, residual, ldr, workspace, ws_bytes, 0, stream);
}

extern "C" int hap_grouped_gemm_bf16_sms(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                                         int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                                         const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                                         int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                                         void* workspace, size_t ws_bytes, int32_t sm_budget, void* stream) {
  using namespace hap::gemm;
  if (!A || !B || !C || a_rows < 0 || K <= 0 || N <= 0 || n_groups <= 0 || sm_budget < 0) return HAP_ERR_INVALID_ARG;
  if (!seg) n_segs = 1;
  if (n_segs <= 0 || n_segs > kMaxSegs) return HAP_ERR_INVALID_ARG;
  if (!seg_group && n_segs != n_groups && seg) return HAP_ERR_INVALID_ARG;
  if (!seg && n_groups != 1) return HAP_ERR_INVALID_ARG;
  if (a_rows > INT32_MAX || N * n_groups > INT32_MAX || K > INT32_MAX) return HAP_ERR_UNSUPPORTED;
  if (K % 8 || lda % 8 || ldc % 8 || N % 8 || lda < K) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return HAP_ERR_MISALIGNED;
  if (a_rows == 0) return HAP_OK;
  Params p{};
  p.a_rows = (int32_t)a_rows;
  p.K = (int32_t)K;
  p.N = (int32_t)N;
  p.n_segs = (int32_t)n_segs;
  p.seg_group = seg_group;
  p.epi = epilogue;
  p.seg = seg;
  p.C = reinterpret_cast<__nv_bfloat16*>(C);
  p.ldc = ldc;
  p.sms = sm_budget < kNumSMs ? sm_budget : 0;
  if (epilogue == HAP_EPI_SWIGLU) {
    if (bias || residual) return HAP_ERR_UNSUPPORTED;
    if (swiglu_half <= 0 || swiglu_half > 128 || swiglu_half % 8 || N % (2 * swiglu_half))
      return HAP_ERR_INVALID_ARG;
    p.hw = (int32_t)swiglu_half;
    p.BN = (int32_t)(2 * swiglu_half);
    if (p.BN % 16) return HAP_ERR_UNSUPPORTED;
    p.out_cols = (int32_t)(N / 2);
    if (ldc < p.out_cols) return HAP_ERR_INVALID_ARG;
  } else if (epilogue == HAP_EPI_STORE) {
    p.BN = pick_bn(N);
    p.out_cols = (int32_t)N;
    if (ldc < N) return HAP_ERR_INVALID_ARG;
    if (residual && (ldr % 8 || ldr < N || (reinterpret_cast<uintptr_t>(residual) & 15))) return HAP_ERR_MISALIGNED;
    if (bias && (reinterpret_cast<uintptr_t>(bias) & 15)) return HAP_ERR_MISALIGNED;
    p.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
    p.resid = reinterpret_cast<const __nv_bfloat16*>(residual);
    p.ldr = ldr;
  } else if (epilogue == HAP_EPI_F32) {
    // raw fp32 accumulators (no bias / residual / rounding): C is float
    // [a_rows, N] dense (ldc == N); never split (one K pass per element)
    if (bias || residual || ldc != N) return HAP_ERR_UNSUPPORTED;
    if (reinterpret_cast<uintptr_t>(C) & 15) return HAP_ERR_MISALIGNED;
    p.BN = pick_bn(N);
    p.out_cols = (int32_t)N;
    p.part = reinterpret_cast<float*>(C);
    return hap::gemm::launch(p, A, a_rows, lda, K, B, n_groups, N, n_segs, nullptr, 0, stream);
  } else {
    return HAP_ERR_INVALID_ARG;
  }

  return hap::gemm::launch(p, A, a_rows, lda, K, B, n_groups, N, n_segs, workspace, ws_bytes, stream);
}

extern "C" int hap_grouped_gemm_bf16_scatter(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                                             int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                                             const int32_t* seg_group, const int64_t* seg_dst,
                                             const int32_t* seg_dst_row0, int64_t ldc, void* stream) {
  using namespace hap::gemm;
  if (!A || !B || !seg || !seg_dst || !seg_dst_row0 || a_rows < 0 || K <= 0 || N <= 0 || n_groups <= 0)
    return HAP_ERR_INVALID_ARG;
  if (n_segs <= 0 || n_segs > kMaxSegs) return HAP_ERR_INVALID_ARG;
  if (!seg_group && n_segs != n_groups) return HAP_ERR_INVALID_ARG;
  if (a_rows > INT32_MAX || N * n_groups > INT32_MAX || K > INT32_MAX) return HAP_ERR_UNSUPPORTED;
  if (K % 8 || lda % 8 || ldc % 8 || N % 8 || lda < K || ldc < N) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return HAP_ERR_MISALIGNED;
  if (a_rows == 0) return HAP_OK;
  Params p{};
  p.a_rows = (int32_t)a_rows;
  p.K = (int32_t)K;
  p.N = (int32_t)N;
  p.n_segs = (int32_t)n_segs;
  p.seg = seg;
  p.seg_group = seg_group;
  p.epi = HAP_EPI_STORE;
  p.BN = pick_bn(N);
  p.out_cols = (int32_t)N;
  p.ldc = ldc;
  p.seg_dst = seg_dst;
  p.seg_dst_row0 = seg_dst_row0;
  // no split-K workspace: the slice reduce writes through C only
  return hap::gemm::launch(p, A, a_rows, lda, K, B, n_groups, N, n_segs, nullptr, 0, stream);
}

extern "C" int hap_grouped_gemm_bf16(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                                     int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                                     const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                                     int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                                     void* stream) {
  return hap_grouped_gemm_bf16_ex(A, a_rows, lda, K, B, n_groups, N, seg, n_segs, seg_group, C, ldc, epilogue,
                                  swiglu_half, bias, residual, ldr, nullptr, 0, stream);
}

extern "C" int hap_gemm_qkv_rope_ex(const void* A, int64_t M, int64_t lda, int64_t K, const void* W, int64_t N,
                                    const void* bias, void* C, int64_t ldc, const int32_t* positions,
                                    int64_t n_rope_heads, int64_t head_dim, float theta, void* workspace,
                                    size_t ws_bytes, void* stream) {
  using namespace hap::gemm;
  if (!A || !W || !C || !positions || M < 0 || K <= 0 || N <= 0) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  if (N % head_dim || n_rope_heads < 0 || n_rope_heads * head_dim > N) return HAP_ERR_INVALID_ARG;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return HAP_ERR_UNSUPPORTED;
  if (K % 8 || lda % 8 || ldc % 8 || lda < K || ldc < N) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(C)) & 15)
    return HAP_ERR_MISALIGNED;
  if (M == 0) return HAP_OK;
  Params p{};
  p.a_rows = (int32_t)M;
  p.K = (int32_t)K;
  p.N = (int32_t)N;
  p.n_segs = 1;
  p.epi = kEpiRope;
  p.C = reinterpret_cast<__nv_bfloat16*>(C);
  p.ldc = ldc;
  p.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
  p.positions = positions;
  p.head_dim = (int32_t)head_dim;
  p.rope_cols = (int32_t)(n_rope_heads * head_dim);
  p.theta = theta;
  p.out_cols = (int32_t)N;
  // whole heads per tile: largest multiple of head_dim <= 256 dividing N
  p.BN = (int32_t)head_dim;
  for (int bn = 256; bn >= head_dim; bn -= (int)head_dim)
    if (N % bn == 0) { p.BN = bn; break; }
  return launch(p, A, M, lda, K, W, 1, N, 1, workspace, ws_bytes, stream);
}

extern "C" int hap_rmsnorm_gemm_qkv_rope(const void* x, int64_t M, int64_t ldx, int64_t K, const void* norm_w,
                                         float eps, void* hn, int64_t ldhn, const void* W, int64_t N,
                                         const void* bias, void* C, int64_t ldc, const int32_t* positions,
                                         int64_t n_rope_heads, int64_t head_dim, float theta, void* workspace,
                                         size_t ws_bytes, void* stream) {
  using namespace hap::gemm;
  if (!x || !norm_w || !hn || !W || !C || !positions || M < 0 || K <= 0 || N <= 0) return HAP_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return HAP_ERR_UNSUPPORTED;
  if (N % head_dim || n_rope_heads < 0 || n_rope_heads * head_dim > N) return HAP_ERR_INVALID_ARG;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return HAP_ERR_UNSUPPORTED;
  if (K % 8 || ldx % 8 || ldhn % 8 || ldc % 8 || ldx < K || ldhn < K || ldc < N) return HAP_ERR_MISALIGNED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(norm_w) | reinterpret_cast<uintptr_t>(hn) |
       reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(C)) & 15)
    return HAP_ERR_MISALIGNED;
  if (M == 0) return HAP_OK;
  // the GEMV path (1-2 rows, decode) normalises while staging its rows: one launch
  if (gemv_mode() > 0 && M <= kGvAutoRows && N % 2 == 0 && M * K * 2 <= 192 * 1024 &&
      N * K * 2 <= (int64_t)64 << 20) {
    Params p{};
    p.a_rows = (int32_t)M;
    p.K = (int32_t)K;
    p.N = (int32_t)N;
    p.n_segs = 1;
    p.epi = kEpiRope;
    p.C = reinterpret_cast<__nv_bfloat16*>(C);
    p.ldc = ldc;
    p.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
    p.positions = positions;
    p.head_dim = (int32_t)head_dim;
    p.rope_cols = (int32_t)(n_rope_heads * head_dim);
    p.theta = theta;
    p.out_cols = (int32_t)N;
    p.norm_w = reinterpret_cast<const __nv_bfloat16*>(norm_w);
    p.norm_eps = eps;
    return launch_gemv(p, x, ldx, W, stream);
  }
  const int st = hap_rmsnorm(x, M, K, ldx, norm_w, eps, hn, ldhn, stream);
  if (st != HAP_OK) return st;
  return hap_gemm_qkv_rope_ex(hn, M, ldhn, K, W, N, bias, C, ldc, positions, n_rope_heads, head_dim, theta, workspace,
                              ws_bytes, stream);
}

extern "C" int hap_gemm_qkv_rope(const void* A, int64_t M, int64_t lda, int64_t K, const void* W, int64_t N,
                                 const void* bias, void* C, int64_t ldc, const int32_t* positions,
                                 int64_t n_rope_heads, int64_t head_dim, float theta, void* stream) {
  return hap_gemm_qkv_rope_ex(A, M, lda, K, W, N, bias, C, ldc, positions, n_rope_heads, head_dim, theta, nullptr,
                              0, stream);
}
