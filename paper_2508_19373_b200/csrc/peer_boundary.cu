// Device-side pieces of the DP<->TP boundary over peer memory (SURVEY §8(e)
// fusions 2-3): the boundary AllGather is pushed by the RMSNorm that produces
// the rows (hap_rmsnorm_multi), the expert-TP ReduceScatter by the combine
// that produces the partial sums (hap_moe_combine_chunked); these two kernels
// close each exchange without the host:
//
//   hap_peer_barrier   one CTA: system fence, publish the next epoch into
//                      every rank's flag slot for this rank, wait until every
//                      rank published it.  Epochs only grow, so one flag row
//                      per group serves every barrier of every call, and the
//                      epoch lives in device memory (CUDA-graph capturable).
//   hap_reduce_slots   owner side of the ReduceScatter: out = sum over the
//                      n_slots pushed partials in slot (= rank) order, fp32,
//                      one bf16 rounding — identical bytes for any arrival
//                      order.
//
// Replaces: the boundary AllGather + ReduceScatter pair of comm_volume
// (reference strategies.py:324-332) and the expert-TP reduction
// (strategies.py:341-342) as NCCL calls.
#include "common.cuh"

namespace hap {
namespace peer_bd {

constexpr int kThreads = 256;

__global__ void barrier_kernel(const int64_t* __restrict__ sig_tab, int32_t* __restrict__ epoch, int n_ranks,
                               int rank) {
  pdl_wait();  // every earlier kernel of this stream (the pushes) has completed
  if (threadIdx.x != 0) return;
  const int32_t e = epoch[0] + 1;
  __threadfence_system();  // this rank's earlier stores (previous kernels) before the flag
  for (int p = 0; p < n_ranks; ++p) st_release_sys(reinterpret_cast<int32_t*>(sig_tab[p]) + rank, e);
  const int32_t* mine = reinterpret_cast<const int32_t*>(sig_tab[rank]);
  for (int p = 0; p < n_ranks; ++p) wait_flag_sys(mine + p, e);
  epoch[0] = e;
}

__global__ void __launch_bounds__(kThreads) reduce_slots_kernel(const uint4* __restrict__ slots, int n_slots,
                                                                int64_t nv, uint4* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nv; i += (int64_t)gridDim.x * kThreads) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    for (int s = 0; s < n_slots; ++s) {
      const uint4 v = __ldcv(slots + (int64_t)s * nv + i);  // written by peers: bypass L1
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    out[i] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                        pack_bf16x2(acc[6], acc[7]));
  }
}

// Copy `n` int32 from src to dst_tab[p] + off (bytes) for every p: tiny
// all-gather pushes (the EP segment offsets).
__global__ void broadcast_i32_kernel(const int32_t* __restrict__ src, int n, const int64_t* __restrict__ dst_tab,
                                     int n_dst, int64_t off) {
  pdl_wait();
  for (int p = blockIdx.x; p < n_dst; p += gridDim.x) {
    int32_t* d = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(dst_tab[p]) + off);
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = src[i];
  }
}

// EP exchange plan from the gathered segment offsets segs[s][0..E] of every
// source s (rows of source s for global expert e: C[s][e] = segs[s][e+1] -
// segs[s][e]); expert e lives on EP rank e / El.  Destination d receives
// blocks (s, j) in lexicographic order, block (s, j) = C[s][d*El + j] rows.
//   dst_row0[e]        (int64) row of my segment e in rank e/El's receive buffer
//   seg_r[0..ep*El]    (int32) my receive blocks' offsets (the GEMM segments)
//   seg_dst_row0[b]    (int32) for my block b = (s, j): row of source s's
//                      x_perm segment of expert me*El + j (combine target)
__global__ void ep_plan_kernel(const int32_t* __restrict__ segs, int ep, int El, int me, int64_t* __restrict__ dst_row0,
                               int32_t* __restrict__ seg_r, int32_t* __restrict__ seg_dst_row0) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const int E = ep * El;
  auto C = [&](int s, int e) { return segs[s * (E + 1) + e + 1] - segs[s * (E + 1) + e]; };
  for (int e = 0; e < E; ++e) {  // blocks (s, j) < (me, e % El) at destination d = e / El
    const int d = e / El;
    int64_t off = 0;
    for (int s = 0; s < me; ++s)
      for (int j = 0; j < El; ++j) off += C(s, d * El + j);
    for (int j = 0; j < e % El; ++j) off += C(me, d * El + j);
    dst_row0[e] = off;
  }
  int32_t acc = 0;
  for (int s = 0; s < ep; ++s)
    for (int j = 0; j < El; ++j) {
      seg_r[s * El + j] = acc;
      acc += C(s, me * El + j);
      seg_dst_row0[s * El + j] = segs[s * (E + 1) + me * El + j];
    }
  seg_r[E] = acc;
}

}  // namespace peer_bd
}  // namespace hap

extern "C" int hap_peer_barrier(const int64_t* sig_tab, int32_t* epoch, int32_t n_ranks, int32_t rank, void* stream) {
  using namespace hap::peer_bd;
  if (!sig_tab || !epoch || n_ranks < 1 || rank < 0 || rank >= n_ranks) return HAP_ERR_INVALID_ARG;
  if (hap::launch_k(barrier_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), sig_tab, epoch,
                    (int)n_ranks, (int)rank) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_reduce_slots_bf16(const void* slots, int64_t n_slots, int64_t rows, int64_t h, void* out,
                                     void* stream) {
  using namespace hap::peer_bd;
  if (!slots || !out || n_slots < 1 || rows < 0 || h <= 0) return HAP_ERR_INVALID_ARG;
  if (h % 8 || ((reinterpret_cast<uintptr_t>(slots) | reinterpret_cast<uintptr_t>(out)) & 15))
    return HAP_ERR_MISALIGNED;
  const int64_t nv = rows * h / 8;
  if (nv == 0) return HAP_OK;
  int64_t grid = (nv + kThreads - 1) / kThreads;
  if (grid > 148 * 8) grid = 148 * 8;
  if (hap::launch_k(reduce_slots_kernel, dim3((unsigned)grid), dim3(kThreads), 0,
                    reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const uint4*>(slots), (int)n_slots, nv,
                    reinterpret_cast<uint4*>(out)) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_peer_broadcast_i32(const int32_t* src, int64_t n, const int64_t* dst_tab, int32_t n_dst,
                                      int64_t dst_offset_bytes, void* stream) {
  using namespace hap::peer_bd;
  if (!src || !dst_tab || n < 0 || n_dst < 1 || dst_offset_bytes < 0 || (dst_offset_bytes & 3))
    return HAP_ERR_INVALID_ARG;
  if (n == 0) return HAP_OK;
  if (hap::launch_k(broadcast_i32_kernel, dim3((unsigned)n_dst), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream),
                    src, (int)n, dst_tab, (int)n_dst, dst_offset_bytes) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}

extern "C" int hap_ep_exchange_plan(const int32_t* segs, int32_t ep, int32_t experts_local, int32_t me,
                                    int64_t* dst_row0, int32_t* seg_r, int32_t* seg_dst_row0, void* stream) {
  using namespace hap::peer_bd;
  if (!segs || !dst_row0 || !seg_r || !seg_dst_row0 || ep < 1 || experts_local < 1 || me < 0 || me >= ep)
    return HAP_ERR_INVALID_ARG;
  if (hap::launch_k(ep_plan_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), segs, (int)ep,
                    (int)experts_local, (int)me, dst_row0, seg_r, seg_dst_row0) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
