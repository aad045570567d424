// One-shot all-reduce over peer-mapped memory for decode-size messages
// (SURVEY §8(e) fusion 1: the attention-TP / expert-TP AllReduce of a decode
// step is 0.5 MB at Mixtral B=64, latency- not bandwidth-bound).
//
// Every rank owns a symmetric region: data[2][n_max] bf16 (double-buffered by
// call parity) and sig[n_ctas][n_ranks] int32 flags; each rank keeps a local
// epoch[n_ctas].  CTA c of rank r, call e:
//   1. copies its slice of the input into data_r[e & 1],
//   2. publishes flag e into sig_p[c][r] of every rank p (system-scope
//      release after a system fence),
//   3. waits until sig_r[c][p] >= e for every p (system-scope acquire),
//   4. sums slice c of data_p[e & 1] over p = 0..N-1 in rank order (fp32,
//      one bf16 rounding) -> identical bytes on every rank.
// CTA c only reads what CTA c of each peer wrote, so the per-CTA flags are the
// whole barrier; parity double buffering + the next call's barrier keep a fast
// rank from overwriting data a slow peer is still reading.  No host work, so the
// kernel is CUDA-graph capturable.  A launch may play several ranks
// (grid.y = ranks_in_launch, rank = rank0 + blockIdx.y) — the single-GPU
// validation runs all ranks in one launch, their CTAs co-resident.
//
// Replaces: the AllReduce rows of comm_volume (reference strategies.py:314-322,
// 341-342) on the decode path.
#include "common.cuh"

namespace hap {
namespace peer_ar {

constexpr int kThreads = 256;


__global__ void __launch_bounds__(kThreads) allreduce_kernel(const int64_t* __restrict__ in_ptrs,
                                                             const int64_t* __restrict__ out_ptrs,
                                                             const int64_t* __restrict__ epoch_ptrs,
                                                             const int64_t* __restrict__ data_ptrs,
                                                             const int64_t* __restrict__ sig_ptrs, int64_t n,
                                                             int64_t n_max, int n_ranks, int rank0) {
  pdl_trigger();
  pdl_wait();
  __shared__ int32_t e_s;
  const int r = rank0 + blockIdx.y;
  const int c = blockIdx.x, n_ctas = gridDim.x;
  int32_t* epoch = reinterpret_cast<int32_t*>(epoch_ptrs[r]);
  if (threadIdx.x == 0) e_s = epoch[c] + 1;
  __syncthreads();
  const int32_t e = e_s;
  const int par = e & 1;
  // 16-byte vectors; slice of CTA c
  const int64_t nv = n / 8;
  const int64_t per = (nv + n_ctas - 1) / n_ctas;
  const int64_t v0 = c * per, v1 = min(nv, v0 + per);
  const uint4* in = reinterpret_cast<const uint4*>(in_ptrs[r]);
  uint4* mine = reinterpret_cast<uint4*>(data_ptrs[r]) + par * (n_max / 8);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += kThreads) mine[i] = in[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < n_ranks; ++p)
      st_release_sys(reinterpret_cast<int32_t*>(sig_ptrs[p]) + (int64_t)c * n_ranks + r, e);
    const int32_t* my_sig = reinterpret_cast<const int32_t*>(sig_ptrs[r]) + (int64_t)c * n_ranks;
    for (int p = 0; p < n_ranks; ++p) wait_flag_sys(my_sig + p, e);
  }
  __syncthreads();
  uint4* out = reinterpret_cast<uint4*>(out_ptrs[r]);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += kThreads) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    for (int p = 0; p < n_ranks; ++p) {
      const uint4 v = __ldcv(reinterpret_cast<const uint4*>(data_ptrs[p]) + par * (n_max / 8) + i);
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
  if (threadIdx.x == 0) epoch[c] = e;
}

}  // namespace peer_ar
}  // namespace hap

extern "C" size_t hap_peer_allreduce_sig_bytes(int32_t n_ranks, int32_t n_ctas) {
  if (n_ranks < 1 || n_ctas < 1) return 0;
  return (size_t)n_ranks * n_ctas * sizeof(int32_t);
}

extern "C" int hap_peer_allreduce_bf16(const int64_t* in_ptrs, const int64_t* out_ptrs, const int64_t* epoch_ptrs,
                                       const int64_t* data_ptrs, const int64_t* sig_ptrs, int64_t n, int64_t n_max,
                                       int32_t n_ranks, int32_t rank0, int32_t ranks_in_launch, int32_t n_ctas,
                                       void* stream) {
  using namespace hap::peer_ar;
  if (!in_ptrs || !out_ptrs || !epoch_ptrs || !data_ptrs || !sig_ptrs) return HAP_ERR_INVALID_ARG;
  if (n < 0 || n > n_max || n_ranks < 1 || rank0 < 0 || ranks_in_launch < 1 || rank0 + ranks_in_launch > n_ranks ||
      n_ctas < 1 || n_ctas > 1024)
    return HAP_ERR_INVALID_ARG;
  if (n % 8 || n_max % 8) return HAP_ERR_MISALIGNED;
  if (n == 0) return HAP_OK;
  { if (hap::launch_k(allreduce_kernel, dim3((unsigned)n_ctas, (unsigned)ranks_in_launch), dim3(kThreads), 0,
                      reinterpret_cast<cudaStream_t>(stream), in_ptrs, out_ptrs, epoch_ptrs, data_ptrs, sig_ptrs, n,
                      n_max, (int)n_ranks, (int)rank0) != cudaSuccess) return HAP_ERR_LAUNCH; }
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
