// Batched 2-D strided copy: many (src, dst, rows, row_bytes, pitches) pieces in
// one launch.  Used by the prefill->decode expert reshard (reference
// transition.py:153-177, Eq.6 T_reshard): the pack phase gathers the
// (unit, TP-slice) pieces other ranks need straight out of the packed
// interleaved gate/up and [h, I] down tensors, the unpack phase scatters the
// received pieces straight into the destination packing.  Each piece is a
// handful of 2-D blocks (gate / up: n/hw SwiGLU blocks of hw*h contiguous
// elements; down: h rows of `per` columns), so one descriptor per block.
//
// HBM-bound byte movement (2 bytes of traffic per byte moved).  The work is
// cut into 16 KB chunks: a segment of one long row, or whole rows of a short-
// row record (the down pieces' rows are only `per` columns, 3.5 KB at Mixtral
// TP 8, so one row per chunk would leave most lanes idle); the host computes
// each descriptor's first chunk index, a persistent grid (CTAs on every SM)
// strides over the chunks, each thread issues its four 16-byte streaming
// loads before any store.  Descriptors travel by value in the
// kernel parameter block (no device workspace, graph capturable).
#include "common.cuh"

namespace hap {
namespace copy2d {

constexpr int kThreads = 256;
constexpr int kVec = 4;                                // 16-byte vectors in flight per thread
constexpr int64_t kChunk = (int64_t)kThreads * kVec * 16;  // 16 KB
constexpr int kMaxDescs = 192;                         // per launch: 192 * 72 B + header < 16 KB of params

struct Desc {
  const char* src;
  char* dst;
  int64_t rows, row_bytes, src_pitch, dst_pitch;
  int64_t chunks_per_row;  // long rows (>= half a chunk): segments per row; else 0
  int64_t rows_per_chunk;  // short rows: whole rows per chunk
};

struct Batch {
  int n;
  int64_t total;
  int64_t first[kMaxDescs];  // exclusive prefix of rows * chunks_per_row
  Desc d[kMaxDescs];
};

__global__ void __launch_bounds__(kThreads) copy2d_kernel(const __grid_constant__ Batch b) {
  pdl_trigger();
  pdl_wait();
  for (int64_t c = blockIdx.x; c < b.total; c += gridDim.x) {
    int lo = 0, hi = b.n - 1;  // last descriptor with first <= c
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (b.first[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const Desc& d = b.d[lo];
    const int64_t local = c - b.first[lo];
    uint4 v[kVec];
    if (d.chunks_per_row) {  // one segment of a long row
      const int64_t row = local / d.chunks_per_row;
      const int64_t off = (local - row * d.chunks_per_row) * kChunk;
      const int64_t len = min(kChunk, d.row_bytes - off);
      const uint4* s = reinterpret_cast<const uint4*>(d.src + row * d.src_pitch + off);
      uint4* t = reinterpret_cast<uint4*>(d.dst + row * d.dst_pitch + off);
      const int n16 = (int)(len >> 4);
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int j = i * kThreads + threadIdx.x;
        if (j < n16) v[i] = __ldcs(s + j);
      }
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int j = i * kThreads + threadIdx.x;
        if (j < n16) __stcs(t + j, v[i]);
      }
    } else {  // whole short rows: vector j of the chunk is (row j / vpr, column j % vpr)
      const int64_t row0 = local * d.rows_per_chunk;
      const int64_t nr = min(d.rows_per_chunk, d.rows - row0);
      const int vpr = (int)(d.row_bytes >> 4);
      const int n16 = (int)nr * vpr;
      const char* s = d.src + row0 * d.src_pitch;
      char* t = d.dst + row0 * d.dst_pitch;
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int j = i * kThreads + threadIdx.x;
        if (j < n16) {
          const int r = j / vpr, col = j - r * vpr;
          v[i] = __ldcs(reinterpret_cast<const uint4*>(s + r * d.src_pitch) + col);
        }
      }
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int j = i * kThreads + threadIdx.x;
        if (j < n16) {
          const int r = j / vpr, col = j - r * vpr;
          __stcs(reinterpret_cast<uint4*>(t + r * d.dst_pitch) + col, v[i]);
        }
      }
    }
  }
}

}  // namespace copy2d
}  // namespace hap

extern "C" int hap_copy2d_batched(const int64_t* descs, int64_t n_descs, void* stream) {
  using namespace hap::copy2d;
  if (n_descs < 0 || (n_descs > 0 && !descs)) return HAP_ERR_INVALID_ARG;
  // validate everything before the first launch
  for (int64_t i = 0; i < n_descs; ++i) {
    const int64_t* e = descs + 6 * i;
    const int64_t src = e[0], dst = e[1], rows = e[2], row_bytes = e[3], sp = e[4], dp = e[5];
    if (rows < 0 || row_bytes < 0) return HAP_ERR_INVALID_ARG;
    if (rows == 0 || row_bytes == 0) continue;
    if (!src || !dst || (rows > 1 && (sp < row_bytes || dp < row_bytes))) return HAP_ERR_INVALID_ARG;
    if ((src | dst | row_bytes | (rows > 1 ? (sp | dp) : 0)) & 15) return HAP_ERR_MISALIGNED;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Batch b;
  int64_t i = 0;
  while (i < n_descs) {
    b.n = 0;
    b.total = 0;
    for (; i < n_descs && b.n < kMaxDescs; ++i) {
      const int64_t* e = descs + 6 * i;
      if (e[2] == 0 || e[3] == 0) continue;
      Desc& d = b.d[b.n];
      d.src = reinterpret_cast<const char*>(e[0]);
      d.dst = reinterpret_cast<char*>(e[1]);
      d.rows = e[2];
      d.row_bytes = e[3];
      d.src_pitch = e[4];
      d.dst_pitch = e[5];
      b.first[b.n] = b.total;
      if (e[3] * 2 > kChunk) {
        d.chunks_per_row = (e[3] + kChunk - 1) / kChunk;
        d.rows_per_chunk = 1;
        b.total += e[2] * d.chunks_per_row;
      } else {
        d.chunks_per_row = 0;
        d.rows_per_chunk = kChunk / e[3];
        b.total += (e[2] + d.rows_per_chunk - 1) / d.rows_per_chunk;
      }
      ++b.n;
    }
    if (b.n == 0) continue;
    const int64_t grid = b.total < 148 * 8 ? b.total : 148 * 8;
    if (hap::launch_k(copy2d_kernel, dim3((unsigned)grid), dim3(kThreads), 0, st, b) != cudaSuccess)
      return HAP_ERR_LAUNCH;
    HAP_CHECK_LAUNCH();
  }
  return HAP_OK;
}
