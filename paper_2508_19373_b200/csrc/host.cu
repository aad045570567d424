// Host-side helpers shared by all kernels: TMA descriptor encoding through the
// driver entry point, dynamic shared-memory opt-in, status strings.
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace hap {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

bool encode_tmap_2d_bf16_sw(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                            uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer > 0 ? outer : 1};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// HAP_PDL (experiments; default 0 = off): 1 every launch, 3 decode-size
// launches only (pdl_for).  On every launch it measured +5.6 % on the
// Mixtral-8x7B prefill block (the waiting dependents' smem/TMEM reservations
// cost more than the launch gaps they hide there) and -4..-6 % on the Qwen2-57B
// B=1 decode step before the shared expert moved to a side stream; on the
// current decode graph the row-gated form measures +2 % at Qwen2-57B B=1 and
// ±noise elsewhere (profiles/r02_pdl_ab.txt), so it stays off.
int pdl_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HAP_PDL");
    v = e ? atoi(e) : 0;
  }
  return v;
}
bool pdl_enabled() { return pdl_mode() == 1; }

bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  return encode_tmap_2d_bf16_sw(map, base, inner, outer, row_stride_bytes, box_inner, box_outer, swizzle128 ? 128 : 0);
}

int configure_smem(const void* kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess ? 0 : -1;
}

}  // namespace hap

// Peer mappings of CUDA-IPC buffers are opened by the owner's device guard;
// kernels on this device write through them only with peer access enabled
// from the current device (NVLink P2P).  Idempotent.
extern "C" int hap_enable_peer_access(int peer_device) {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return HAP_ERR_LAUNCH;
  if (peer_device == cur) return HAP_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, cur, peer_device) != cudaSuccess || !can) return HAP_ERR_UNSUPPORTED;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free error state
    return HAP_OK;
  }
  return e == cudaSuccess ? HAP_OK : HAP_ERR_LAUNCH;
}

extern "C" const char* hap_status_string(int status) {
  switch (status) {
    case HAP_OK: return "ok";
    case HAP_ERR_INVALID_ARG: return "invalid argument";
    case HAP_ERR_UNSUPPORTED: return "unsupported shape";
    case HAP_ERR_MISALIGNED: return "misaligned pointer or leading dimension";
    case HAP_ERR_LAUNCH: return "CUDA launch failure";
    case HAP_ERR_WORKSPACE: return "workspace too small";
    case HAP_ERR_DRIVER: return "driver entry point unavailable (cuTensorMapEncodeTiled)";
    default: return "unknown status";
  }
}

extern "C" int hap_abi_version(void) { return 2; }
