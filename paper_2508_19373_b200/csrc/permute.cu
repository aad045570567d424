// Token permute (dispatch re-layout) and weighted combine (unpermute).
//
// Permute is a stable counting sort keyed on the expert id, in three passes:
//   1. rank:    each block takes a contiguous range of rows; per 256-row pass
//               a warp computes stable in-warp ranks with __match_any_sync and
//               per-warp expert counts, combined across warps in row order.
//               Output: local_rank[r] (rank among equal experts inside the
//               block) and block_counts[b][e].
//   2. scan:    per-expert totals -> seg (exclusive prefix), and per-block
//               bases base[b][e] = seg[e] + sum_{b'<b} block_counts[b'][e].
//   3. scatter: dst = base[b(r)][e_r] + local_rank[r]; one warp copies the
//               h-wide bf16 row with 16-byte vector loads/stores.
// Every step is deterministic (no atomics on the ordering path), so the
// permutation is bit-exact against the oracle's stable sort by (expert, row).
//
// Combine reads the k expert outputs of a token (gather), accumulates
// w * y in fp32 in slot order, adds the optional shared-expert output scaled
// by its sigmoid gate and the residual, and rounds once to bf16.
//
// Models: the EP dispatch/combine token re-layout implicit in the all-to-all
// rows of comm_volume (reference strategies.py:334-340).
#include "common.cuh"

namespace hap {
namespace permute {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerBlock = 512;  // 64 blocks at R = 32768 (latency-bound otherwise)
constexpr int kMaxExperts = 512;

struct Workspace {
  int32_t* local_rank;    // [R]
  int32_t* block_counts;  // [NB][E]
  int32_t* block_base;    // [NB][E]
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static size_t ws_bytes(int64_t R, int64_t E, int64_t* nb_out) {
  const int64_t nb = (R + kRowsPerBlock - 1) / kRowsPerBlock;
  if (nb_out) *nb_out = nb;
  return align_up((size_t)R * 4, 256) + 2 * align_up((size_t)(nb > 0 ? nb : 1) * E * 4, 256);
}

__global__ void __launch_bounds__(kThreads) rank_kernel(const int32_t* __restrict__ eid, int R, int E,
                                                        int32_t* __restrict__ local_rank,
                                                        int32_t* __restrict__ block_counts,
                                                        int32_t* __restrict__ block_base, int32_t* __restrict__ seg) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t sm[];
  int32_t* running = sm;             // [E]
  int32_t* warp_cnt = sm + E;        // [kWarps][E]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += kThreads) running[i] = 0;
  const int r_begin = blockIdx.x * kRowsPerBlock;
  const int r_end = min(R, r_begin + kRowsPerBlock);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int base = r_begin; base < r_end; base += kThreads) {
    for (int i = threadIdx.x; i < kWarps * E; i += kThreads) warp_cnt[i] = 0;
    __syncthreads();
    const int r = base + threadIdx.x;
    int e = -1;
    if (r < r_end) {
      e = eid[r];
      if (e < 0 || e >= E) e = -1;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank_in_warp = __popc(peers & lt_mask);
    if (e >= 0 && rank_in_warp == 0) warp_cnt[warp * E + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int off = running[e];
      for (int w2 = 0; w2 < warp; ++w2) off += warp_cnt[w2 * E + e];
      local_rank[r] = off + rank_in_warp;
    } else if (r < r_end) {
      local_rank[r] = -1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E; i += kThreads) {
      int s = 0;
      for (int w2 = 0; w2 < kWarps; ++w2) s += warp_cnt[w2 * E + i];
      running[i] += s;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < E; i += kThreads) block_counts[(int64_t)blockIdx.x * E + i] = running[i];
  if (gridDim.x == 1 && threadIdx.x == 0) {
    // a single block (decode-sized R): the scan is the prefix of its own counts
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      seg[e] = acc;
      block_base[e] = acc;
      acc += running[e];
    }
    seg[E] = acc;
  }
}

__global__ void scan_kernel(const int32_t* __restrict__ block_counts, int NB, int E, int32_t* __restrict__ block_base,
                            int32_t* __restrict__ seg) {
  pdl_trigger();
  pdl_wait();
  __shared__ int32_t totals[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
    for (int b = 0; b < NB; ++b) s += block_counts[(int64_t)b * E + e];
    totals[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      const int c = totals[e];
      totals[e] = acc;
      seg[e] = acc;
      acc += c;
    }
    seg[E] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int acc = totals[e];
    for (int b = 0; b < NB; ++b) {
      block_base[(int64_t)b * E + e] = acc;
      acc += block_counts[(int64_t)b * E + e];
    }
  }
}

__global__ void __launch_bounds__(kThreads) scatter_kernel(const int32_t* __restrict__ eid, int R, int E,
                                                           const int32_t* __restrict__ local_rank,
                                                           const int32_t* __restrict__ block_base,
                                                           const uint4* __restrict__ x, int src_div, int hv,
                                                           uint4* __restrict__ x_out, int32_t* __restrict__ dst_of_row) {
  pdl_trigger();
  pdl_wait();
  const int warp_global = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n_warps = (gridDim.x * kThreads) >> 5;
  for (int r = warp_global; r < R; r += n_warps) {
    int e = eid[r];
    int dst = -1;
    if (e >= 0 && e < E) dst = block_base[(int64_t)(r / kRowsPerBlock) * E + e] + local_rank[r];
    if (lane == 0) dst_of_row[r] = dst;
    if (dst >= 0 && x_out) {
      const uint4* src = x + (int64_t)(r / src_div) * hv;
      uint4* out = x_out + (int64_t)dst * hv;
      int i = lane;
      for (; i + 96 < hv; i += 128) {
        const uint4 a = __ldg(src + i), b = __ldg(src + i + 32), c = __ldg(src + i + 64), d = __ldg(src + i + 96);
        out[i] = a;
        out[i + 32] = b;
        out[i + 64] = c;
        out[i + 96] = d;
      }
      for (; i < hv; i += 32) out[i] = __ldg(src + i);
    }
  }
}

// Decode-size permute (R <= kRowsPerBlock): rank and scatter in ONE launch.
// Every CTA recomputes the stable ranks of all R rows in shared memory (the
// same per-warp __match_any_sync ranks combined in row order as rank_kernel,
// so dst_of_row / seg are identical), CTA 0 writes seg, and the warps of all
// CTAs then copy their rows.  Saves the rank launch on the decode critical
// path; R is at most 512 ids (2 KB), so the redundant ranking is cheap.
__global__ void __launch_bounds__(kThreads) permute_small_kernel(const int32_t* __restrict__ eid, int R, int E,
                                                                 const uint4* __restrict__ x, int src_div, int hv,
                                                                 uint4* __restrict__ x_out,
                                                                 int32_t* __restrict__ dst_of_row,
                                                                 int32_t* __restrict__ seg) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t sm[];
  int32_t* running = sm;                   // [E] -> exclusive bases after the scan
  int32_t* warp_cnt = sm + E;              // [kWarps][E]
  int32_t* rank_s = sm + (1 + kWarps) * E;  // [kRowsPerBlock]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += kThreads) running[i] = 0;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int base = 0; base < R; base += kThreads) {
    for (int i = threadIdx.x; i < kWarps * E; i += kThreads) warp_cnt[i] = 0;
    __syncthreads();
    const int r = base + threadIdx.x;
    int e = -1;
    if (r < R) {
      e = eid[r];
      if (e < 0 || e >= E) e = -1;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank_in_warp = __popc(peers & lt_mask);
    if (e >= 0 && rank_in_warp == 0) warp_cnt[warp * E + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int off = running[e];
      for (int w2 = 0; w2 < warp; ++w2) off += warp_cnt[w2 * E + e];
      rank_s[r] = off + rank_in_warp;
    } else if (r < R) {
      rank_s[r] = -1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E; i += kThreads) {
      int s2 = 0;
      for (int w2 = 0; w2 < kWarps; ++w2) s2 += warp_cnt[w2 * E + i];
      running[i] += s2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // counts -> exclusive bases (and seg from CTA 0)
    int acc = 0;
    for (int e2 = 0; e2 < E; ++e2) {
      const int c = running[e2];
      running[e2] = acc;
      if (blockIdx.x == 0) seg[e2] = acc;
      acc += c;
    }
    if (blockIdx.x == 0) seg[E] = acc;
  }
  __syncthreads();
  const int n_warps = (gridDim.x * kThreads) >> 5;
  for (int r = (blockIdx.x * kThreads + threadIdx.x) >> 5; r < R; r += n_warps) {
    const int e2 = eid[r];
    const int dst = (e2 >= 0 && e2 < E) ? running[e2] + rank_s[r] : -1;
    if (lane == 0) dst_of_row[r] = dst;
    if (dst >= 0 && x_out) {
      const uint4* src = x + (int64_t)(r / src_div) * hv;
      uint4* out = x_out + (int64_t)dst * hv;
      int i = lane;
      for (; i + 96 < hv; i += 128) {
        const uint4 a = __ldg(src + i), b = __ldg(src + i + 32), c = __ldg(src + i + 64), d = __ldg(src + i + 96);
        out[i] = a;
        out[i + 32] = b;
        out[i + 64] = c;
        out[i + 96] = d;
      }
      for (; i < hv; i += 32) out[i] = __ldg(src + i);
    }
  }
}

// Large-T combine: one warp per token row; the k slot rows / weights are read
// once per token and every lane streams its 16-byte column chunks of the k
// expert outputs (+ shared output, + residual) with 4 chunks in flight, so a
// warp keeps several KB of loads outstanding instead of one dependent pair per
// 256-column item.  Same accumulation order as combine_kernel (slot order,
// then shared, then residual; fp32; one bf16 rounding): bit-identical.
constexpr int kCombineU = 4;

// Output row of token t: out + t*hv, or (out_tab != nullptr, the reduce-scatter
// push of hap_moe_combine_chunked) row (slot*chunk_rows + t % chunk_rows) of
// the buffer out_tab[t / chunk_rows] — chunk q of the partial sums goes
// straight into slot `slot` of its owner q's (peer-mapped) receive buffer.
__device__ __forceinline__ uint4* combine_out_row(uint4* out, const int64_t* __restrict__ out_tab, int chunk_rows,
                                                  int slot, int t, int hv) {
  if (out_tab == nullptr) return out + (int64_t)t * hv;
  return reinterpret_cast<uint4*>(__ldg(out_tab + t / chunk_rows)) +
         ((int64_t)slot * chunk_rows + t % chunk_rows) * hv;
}
__global__ void __launch_bounds__(kThreads) combine_row_kernel(const uint4* __restrict__ y, const int32_t* __restrict__ dst,
                                                               const float* __restrict__ tw, int T, int k, int hv,
                                                               const uint4* __restrict__ resid, int res_row0,
                                                               int res_rows, const uint4* __restrict__ shared_y,
                                                               const float* __restrict__ shared_gate,
                                                               uint4* __restrict__ out, const int64_t* __restrict__ out_tab,
                                                            int chunk_rows, int slot) {
  pdl_trigger();
  pdl_wait();
  const int warp_global = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n_warps = (gridDim.x * kThreads) >> 5;
  for (int t = warp_global; t < T; t += n_warps) {
    const int my_row = lane < k ? dst[(int64_t)t * k + lane] : -1;
    const float my_w = lane < k ? tw[(int64_t)t * k + lane] : 0.f;
    const float sg = shared_y ? shared_gate[t] : 0.f;
    const bool has_res = resid && t >= res_row0 && t < res_row0 + res_rows;
    for (int c0 = lane; c0 < hv; c0 += 32 * kCombineU) {
      float acc[kCombineU][8];
#pragma unroll
      for (int u = 0; u < kCombineU; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
      for (int j = 0; j < k; ++j) {
        const int row = __shfl_sync(0xffffffffu, my_row, j);
        const float wj = __shfl_sync(0xffffffffu, my_w, j);
        if (row < 0) continue;
        uint4 v[kCombineU];
#pragma unroll
        for (int u = 0; u < kCombineU; ++u) {
          const int c = c0 + 32 * u;
          v[u] = c < hv ? __ldg(y + (int64_t)row * hv + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kCombineU; ++u) {
          const uint32_t vw[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16x2(vw[i]);
            acc[u][2 * i] = fmaf(wj, f.x, acc[u][2 * i]);
            acc[u][2 * i + 1] = fmaf(wj, f.y, acc[u][2 * i + 1]);
          }
        }
      }
      if (shared_y) {
#pragma unroll
        for (int u = 0; u < kCombineU; ++u) {
          const int c = c0 + 32 * u;
          if (c >= hv) continue;
          const uint4 v = __ldg(shared_y + (int64_t)t * hv + c);
          const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16x2(vw[i]);
            acc[u][2 * i] = fmaf(sg, f.x, acc[u][2 * i]);
            acc[u][2 * i + 1] = fmaf(sg, f.y, acc[u][2 * i + 1]);
          }
        }
      }
      if (has_res) {
#pragma unroll
        for (int u = 0; u < kCombineU; ++u) {
          const int c = c0 + 32 * u;
          if (c >= hv) continue;
          const uint4 v = __ldg(resid + (int64_t)(t - res_row0) * hv + c);
          const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16x2(vw[i]);
            acc[u][2 * i] += f.x;
            acc[u][2 * i + 1] += f.y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCombineU; ++u) {
        const int c = c0 + 32 * u;
        if (c < hv)
          combine_out_row(out, out_tab, chunk_rows, slot, t, hv)[c] = make_uint4(pack_bf16x2(acc[u][0], acc[u][1]), pack_bf16x2(acc[u][2], acc[u][3]),
                                                pack_bf16x2(acc[u][4], acc[u][5]), pack_bf16x2(acc[u][6], acc[u][7]));
      }
    }
  }
}

// One warp per (token, 256-column chunk): lane owns columns chunk*256 + lane*8
// .. +8.  Slot rows/weights are loaded once per warp (lane j holds slot j) and
// broadcast with shuffles, so small-T (decode) calls still fill the GPU.
__global__ void __launch_bounds__(kThreads) combine_kernel(const uint4* __restrict__ y, const int32_t* __restrict__ dst,
                                                           const float* __restrict__ tw, int T, int k, int hv,
                                                           const uint4* __restrict__ resid, int res_row0,
                                                           int res_rows, const uint4* __restrict__ shared_y,
                                                           const float* __restrict__ shared_gate,
                                                           uint4* __restrict__ out, const int64_t* __restrict__ out_tab,
                                                            int chunk_rows, int slot) {
  pdl_trigger();
  pdl_wait();
  const int warp_global = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n_warps = (gridDim.x * kThreads) >> 5;
  const int n_chunks = (hv + 31) / 32;
  for (int item = warp_global; item < T * n_chunks; item += n_warps) {
    const int t = item / n_chunks;
    const int c = (item % n_chunks) * 32 + lane;
    const int my_row = lane < k ? dst[(int64_t)t * k + lane] : -1;
    const float my_w = lane < k ? tw[(int64_t)t * k + lane] : 0.f;
    const bool ok = c < hv;  // all lanes stay for the shuffles below
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int j = 0; j < k; ++j) {
      const int row = __shfl_sync(0xffffffffu, my_row, j);
      const float wj = __shfl_sync(0xffffffffu, my_w, j);
      if (row < 0 || !ok) continue;
      const uint4 v = __ldg(y + (int64_t)row * hv + c);
      const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(vw[i]);
        acc[2 * i] = fmaf(wj, f.x, acc[2 * i]);
        acc[2 * i + 1] = fmaf(wj, f.y, acc[2 * i + 1]);
      }
    }
    if (!ok) continue;
    if (shared_y) {
      const float sg = shared_gate[t];
      const uint4 v = __ldg(shared_y + (int64_t)t * hv + c);
      const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(vw[i]);
        acc[2 * i] = fmaf(sg, f.x, acc[2 * i]);
        acc[2 * i + 1] = fmaf(sg, f.y, acc[2 * i + 1]);
      }
    }
    if (resid && t >= res_row0 && t < res_row0 + res_rows) {
      const uint4 v = __ldg(resid + (int64_t)(t - res_row0) * hv + c);
      const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16x2(vw[i]);
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
      }
    }
    combine_out_row(out, out_tab, chunk_rows, slot, t, hv)[c] =
        make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                   pack_bf16x2(acc[6], acc[7]));
  }
}

// EP dispatch over peer memory: rows [seg[s], seg[s+1]) of src go to
// dst_base[s] + (dst_row0[s] + i) * ldd (dst_base[s] may be a peer-mapped
// address, so the stores travel over NVLink).  One warp per row, 16-byte
// vectors, 4 in flight per lane.
__global__ void __launch_bounds__(kThreads) peer_copy_kernel(const uint4* __restrict__ src, int hv, int n_segs,
                                                             const int32_t* __restrict__ seg,
                                                             const int64_t* __restrict__ dst_base,
                                                             const int64_t* __restrict__ dst_row0, int64_t lddv) {
  pdl_trigger();
  pdl_wait();
  const int warp_global = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n_warps = (gridDim.x * kThreads) >> 5;
  const int R = seg[n_segs];
  for (int r = warp_global; r < R; r += n_warps) {
    int lo = 0, hi = n_segs - 1;  // segment of row r: last s with seg[s] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const uint4* in = src + (int64_t)r * hv;
    uint4* out = reinterpret_cast<uint4*>(dst_base[lo]) + (dst_row0[lo] + (r - seg[lo])) * lddv;
    int i = lane;
    for (; i + 96 < hv; i += 128) {
      const uint4 a = __ldg(in + i), b = __ldg(in + i + 32), c = __ldg(in + i + 64), d = __ldg(in + i + 96);
      out[i] = a;
      out[i + 32] = b;
      out[i + 64] = c;
      out[i + 96] = d;
    }
    for (; i < hv; i += 32) out[i] = __ldg(in + i);
  }
}

}  // namespace permute
}  // namespace hap

using namespace hap::permute;

extern "C" size_t hap_moe_permute_workspace_bytes(int64_t R, int64_t n_experts) {
  if (R < 0 || n_experts <= 0) return 0;
  return ws_bytes(R, n_experts, nullptr);
}

// HAP_PERMUTE_SMALL=0 (A/B): decode-size permutes keep the rank + scatter pair
static bool small_permute() {
  static const bool on = [] {
    const char* e = getenv("HAP_PERMUTE_SMALL");
    return !(e && e[0] == '0');
  }();
  return on;
}

extern "C" int hap_moe_permute(const int32_t* expert_of_row, int64_t R, int64_t n_experts, const void* x,
                               int64_t src_row_div, int64_t h, void* x_out, int32_t* dst_of_row, int32_t* seg,
                               void* workspace, size_t ws_size, void* stream) {
  if (!seg || R < 0 || n_experts <= 0) return HAP_ERR_INVALID_ARG;
  if (R > 0 && (!expert_of_row || !dst_of_row)) return HAP_ERR_INVALID_ARG;
  if (n_experts > kMaxExperts || R > INT32_MAX) return HAP_ERR_UNSUPPORTED;
  if (x_out && (!x || src_row_div <= 0 || h <= 0)) return HAP_ERR_INVALID_ARG;
  if (x_out && (h % 8 || ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(x_out)) & 15)))
    return HAP_ERR_MISALIGNED;
  int64_t nb = 0;
  const size_t need = ws_bytes(R, n_experts, &nb);
  if (!workspace || ws_size < need) return HAP_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int E = (int)n_experts;
  uint8_t* w8 = reinterpret_cast<uint8_t*>(workspace);
  int32_t* local_rank = reinterpret_cast<int32_t*>(w8);
  int32_t* block_counts = reinterpret_cast<int32_t*>(w8 + align_up((size_t)R * 4, 256));
  int32_t* block_base =
      reinterpret_cast<int32_t*>(w8 + align_up((size_t)R * 4, 256) + align_up((size_t)(nb > 0 ? nb : 1) * E * 4, 256));
  if (R == 0) {
    cudaMemsetAsync(seg, 0, sizeof(int32_t) * (E + 1), st);
    HAP_CHECK_LAUNCH();
    return HAP_OK;
  }
  if (nb == 1 && small_permute()) {  // decode-size: rank + scatter in one launch
    const int smem_s = (int)(((1 + kWarps) * E + kRowsPerBlock) * sizeof(int32_t));
    int grid_s = (int)((R * 32 + kThreads - 1) / kThreads);
    if (!x_out) grid_s = 1;
    { if (hap::launch_kr(R, permute_small_kernel, dim3(grid_s), dim3(kThreads), smem_s, st, expert_of_row, (int)R, E,
                         reinterpret_cast<const uint4*>(x), (int)(src_row_div > 0 ? src_row_div : 1), (int)(h / 8),
                         reinterpret_cast<uint4*>(x_out), dst_of_row, seg) != cudaSuccess) return HAP_ERR_LAUNCH; }
    HAP_CHECK_LAUNCH();
    return HAP_OK;
  }
  const int smem = (int)((1 + kWarps) * E * sizeof(int32_t));
  { if (hap::launch_kr(R, rank_kernel, dim3((int)nb), dim3(kThreads), smem, st, expert_of_row, (int)R, E, local_rank, block_counts, block_base, seg) != cudaSuccess) return HAP_ERR_LAUNCH; }
  if (nb > 1) {  // one block computes the prefix itself
    { if (hap::launch_kr(R, scan_kernel, dim3(1), dim3(256), 0, st, block_counts, (int)nb, E, block_base, seg) != cudaSuccess) return HAP_ERR_LAUNCH; }
  }
  const int64_t warps_needed = R;
  int grid = (int)((warps_needed * 32 + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  { if (hap::launch_kr(R, scatter_kernel, dim3(grid), dim3(kThreads), 0, st, expert_of_row, (int)R, E, local_rank, block_base,
                                            reinterpret_cast<const uint4*>(x), (int)(src_row_div > 0 ? src_row_div : 1),
                                            (int)(h / 8), reinterpret_cast<uint4*>(x_out), dst_of_row) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

static int combine_launch(const void* y, const int32_t* dst_of_row, const float* topk_w, int64_t T, int64_t k,
                          int64_t h, const void* residual, int64_t res_row0, int64_t res_rows, const void* shared_y,
                          const float* shared_gate, void* out, const int64_t* out_tab, int64_t chunk_rows,
                          int64_t slot, void* stream) {
  if (!y || !dst_of_row || !topk_w || (!out && !out_tab) || T < 0 || k < 1 || k > 32 || h <= 0)
    return HAP_ERR_INVALID_ARG;
  if (h % 8) return HAP_ERR_MISALIGNED;
  if ((shared_y == nullptr) != (shared_gate == nullptr)) return HAP_ERR_INVALID_ARG;
  if (residual && (res_row0 < 0 || res_rows < 0)) return HAP_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(residual) |
       reinterpret_cast<uintptr_t>(shared_y)) & 15)
    return HAP_ERR_MISALIGNED;
  if (T == 0) return HAP_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (T >= 148 * kWarps) {  // enough tokens to fill the GPU with one warp per row
    int grid_r = (int)((T + kWarps - 1) / kWarps);
    if (grid_r > 148 * 16) grid_r = 148 * 16;
    { if (hap::launch_kr(T, combine_row_kernel, dim3(grid_r), dim3(kThreads), 0, st, reinterpret_cast<const uint4*>(y),
                        dst_of_row, topk_w, (int)T, (int)k, (int)(h / 8), reinterpret_cast<const uint4*>(residual),
                        (int)res_row0, (int)res_rows, reinterpret_cast<const uint4*>(shared_y), shared_gate,
                        reinterpret_cast<uint4*>(out), out_tab, (int)chunk_rows, (int)slot) != cudaSuccess) return HAP_ERR_LAUNCH; }
    HAP_CHECK_LAUNCH();
    return HAP_OK;
  }
  const int64_t items = T * ((h / 8 + 31) / 32);
  int grid = (int)((items * 32 + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  { if (hap::launch_kr(T, combine_kernel, dim3(grid), dim3(kThreads), 0, st, reinterpret_cast<const uint4*>(y), dst_of_row, topk_w, (int)T, (int)k,
                                            (int)(h / 8), reinterpret_cast<const uint4*>(residual), (int)res_row0,
                                            (int)res_rows, reinterpret_cast<const uint4*>(shared_y), shared_gate,
                                            reinterpret_cast<uint4*>(out), out_tab, (int)chunk_rows, (int)slot) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_moe_combine(const void* y, const int32_t* dst_of_row, const float* topk_w, int64_t T, int64_t k,
                               int64_t h, const void* residual, int64_t res_row0, int64_t res_rows,
                               const void* shared_y, const float* shared_gate, void* out, void* stream) {
  if (!out) return HAP_ERR_INVALID_ARG;
  return combine_launch(y, dst_of_row, topk_w, T, k, h, residual, res_row0, res_rows, shared_y, shared_gate, out,
                        nullptr, 1, 0, stream);
}

extern "C" int hap_moe_combine_chunked(const void* y, const int32_t* dst_of_row, const float* topk_w, int64_t T,
                                       int64_t k, int64_t h, const void* residual, int64_t res_row0,
                                       int64_t res_rows, const void* shared_y, const float* shared_gate,
                                       const int64_t* out_tab, int64_t chunk_rows, int64_t slot, void* stream) {
  if (!out_tab || chunk_rows < 1 || slot < 0 || T % chunk_rows) return HAP_ERR_INVALID_ARG;
  return combine_launch(y, dst_of_row, topk_w, T, k, h, residual, res_row0, res_rows, shared_y, shared_gate, nullptr,
                        out_tab, chunk_rows, slot, stream);
}

extern "C" int hap_peer_copy_rows(const void* src, int64_t rows_max, int64_t h, const int32_t* seg, int64_t n_segs,
                                  const int64_t* dst_base, const int64_t* dst_row0, int64_t ldd, void* stream) {
  if (!src || !seg || !dst_base || !dst_row0 || rows_max < 0 || h <= 0 || n_segs <= 0) return HAP_ERR_INVALID_ARG;
  if (h % 8 || ldd % 8 || ldd < h || (reinterpret_cast<uintptr_t>(src) & 15)) return HAP_ERR_MISALIGNED;
  if (rows_max == 0) return HAP_OK;
  int grid = (int)((rows_max * 32 + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  { if (hap::launch_k(peer_copy_kernel, dim3(grid), dim3(kThreads), 0, reinterpret_cast<cudaStream_t>(stream),
                      reinterpret_cast<const uint4*>(src), (int)(h / 8), (int)n_segs, seg, dst_base, dst_row0,
                      ldd / 8) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
