// Does a region read by every SM get fetched from DRAM once, or once per die?
// Each of 148 CTAs reads the same `mb` MB region once (16-byte loads, L2
// cached), XORs into a sink.  Run under ncu: dram__bytes_read.sum ~= region
// -> one fetch for the whole chip; ~= 2 x region -> one fetch per die.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void read_same(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[blockIdx.x] = acc;
}
int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 8;
  const size_t n = mb * (1 << 20) / 16;
  uint4 *p, *sink;
  cudaMalloc(&p, n * 16);
  cudaMalloc(&sink, 148 * 16);
  cudaMemset(p, 1, n * 16);
  cudaDeviceSynchronize();
  for (int r = 0; r < 3; ++r) read_same<<<148, 512>>>(p, n, sink);
  cudaDeviceSynchronize();
  printf("done %zu MB\n", mb);
  return 0;
}
