// One-shot all-reduce through NVLink SHARP (NVLS): the in-switch reduction of
// NVSwitch multicast memory (SURVEY §8(e) fusion 1, "NVLS / multimem one-shot
// AllReduce for decode-size messages").
//
// Every rank binds one physical allocation of its own device to a multicast
// object (set up by the caller, peer.NvlsAllReduce); uc_* are this rank's
// unicast view, mc_* the multicast view.  Layout: int32 flag[n_ctas] (one
// counter per CTA), then data[2][n_max] bf16 (double-buffered by call parity).
// CTA c of a call with epoch e:
//   1. copies its slice of `in` into its own data[e & 1] (unicast),
//   2. arrives with one multimem.red.add on flag[c] (the switch adds 1 to
//      flag[c] of every rank) and spins until its own flag[c] >= e * n_ranks,
//   3. reads its slice with multimem.ld_reduce: the switch returns the sum of
//      every rank's data (fp32 accumulation, one bf16 rounding), stored to out.
// The counters only grow, the parity buffers keep a fast rank from
// overwriting data a slow one is still reducing, and nothing touches the host:
// the call is CUDA-graph capturable.
//
// Replaces: the AllReduce rows of comm_volume (reference strategies.py:314-322,
// 341-342) on the decode path, as a switch reduction instead of N-1 peer reads.
#include "common.cuh"

namespace hap {
namespace nvls {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) allreduce_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                             uint8_t* __restrict__ uc, uint8_t* __restrict__ mc,
                                                             int32_t* __restrict__ epoch, int64_t nv,
                                                             int64_t nv_max, int n_ranks, int64_t data_off) {
  pdl_trigger();
  pdl_wait();
  __shared__ int32_t e_s;
  const int c = blockIdx.x, n_ctas = gridDim.x;
  if (threadIdx.x == 0) e_s = epoch[c] + 1;
  __syncthreads();
  const int32_t e = e_s;
  const int64_t per = (nv + n_ctas - 1) / n_ctas;
  const int64_t v0 = c * per, v1 = min(nv, v0 + per);
  uint4* mine = reinterpret_cast<uint4*>(uc + data_off) + (int64_t)(e & 1) * nv_max;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += kThreads) mine[i] = in[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    int32_t* mflag = reinterpret_cast<int32_t*>(mc) + c;
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mflag), "r"(1u) : "memory");
    wait_flag_sys(reinterpret_cast<const int32_t*>(uc) + c, e * n_ranks);
  }
  __syncthreads();
  const uint4* msrc = reinterpret_cast<const uint4*>(mc + data_off) + (int64_t)(e & 1) * nv_max;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += kThreads) {
    uint32_t a, b, c2, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c2), "=r"(d)
                 : "l"(msrc + i)
                 : "memory");
    out[i] = make_uint4(a, b, c2, d);
  }
  if (threadIdx.x == 0) epoch[c] = e;
}

}  // namespace nvls
}  // namespace hap

extern "C" size_t hap_nvls_allreduce_bytes(int64_t n_max, int32_t n_ctas) {
  if (n_max <= 0 || n_max % 8 || n_ctas < 1) return 0;
  const size_t flags = ((size_t)n_ctas * 4 + 4095) / 4096 * 4096;
  return flags + 2 * (size_t)n_max * 2;
}

extern "C" int hap_nvls_allreduce_bf16(const void* in, void* out, void* uc_base, void* mc_base, int32_t* epoch,
                                       int64_t n, int64_t n_max, int32_t n_ranks, int32_t n_ctas, void* stream) {
  using namespace hap::nvls;
  if (!in || !out || !uc_base || !mc_base || !epoch || n < 0 || n > n_max || n_ranks < 1 || n_ctas < 1 ||
      n_ctas > 1024)
    return HAP_ERR_INVALID_ARG;
  if (n % 8 || n_max % 8 ||
      ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(uc_base) |
        reinterpret_cast<uintptr_t>(mc_base)) & 15))
    return HAP_ERR_MISALIGNED;
  if (n == 0) return HAP_OK;
  const int64_t data_off = (int64_t)(((size_t)n_ctas * 4 + 4095) / 4096 * 4096);
  if (hap::launch_k(allreduce_kernel, dim3((unsigned)n_ctas), dim3(kThreads), 0,
                    reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const uint4*>(in),
                    reinterpret_cast<uint4*>(out), reinterpret_cast<uint8_t*>(uc_base),
                    reinterpret_cast<uint8_t*>(mc_base), epoch, n / 8, n_max / 8, (int)n_ranks,
                    data_off) != cudaSuccess)
    return HAP_ERR_LAUNCH;
  HAP_CHECK_LAUNCH();
  return HAP_OK;
}
