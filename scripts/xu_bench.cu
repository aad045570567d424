// Throughput of the softmax instruction mix on one SM (ops / clk / SM): MUFU ex2, cvt.bf16x2,
// ex2.bf16x2, FFMA, max3.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/xu_bench.cu -o /tmp/xu && /tmp/xu
// Measured on B200: ex2.f32 16/clk/SM, cvt.rn.bf16x2.f32 64, ex2.bf16x2 8 pairs, FFMA 121, max3 64.
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

constexpr int ITER = 4096;

template <int MODE>
__global__ void k(float* out, float seed, long long* clk) {
  float a[8];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i) * 1e-6f - 3.f; u[i] = __float_as_uint(a[i]); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // ex2.f32
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (MODE == 1) {  // cvt bf16x2 (pack two fp32)
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        a[i] = __uint_as_float(r) ;
      } else if (MODE == 2) {  // ex2 bf16x2
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      } else if (MODE == 3) {  // 2 ex2 + 1 cvt (softmax mix)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[(i + 4) & 7]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 4) & 7]));
        u[i] ^= r;
      } else if (MODE == 4) {  // FFMA
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      } else if (MODE == 5) {  // cvt f32 -> bf16 single (F2F?)
        uint16_t h;
        asm volatile("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(a[i]));
        u[i] += h;
      } else if (MODE == 6) {  // fmax3
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      } else if (MODE == 7) {  // cvt.rn.f16x2.f32
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        a[i] = __uint_as_float(r);
      } else if (MODE == 8) {  // ex2.approx.f16x2
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int ops_per_inner) {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 148 * 8);
  for (int threads : {256, 512, 1024}) {
    k<MODE><<<148, threads>>>(out, 1.0f, clk);
    k<MODE><<<148, threads>>>(out, 1.0f, clk);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    double ops = (double)threads * ITER * 8 * ops_per_inner;
    printf("%-22s threads=%4d  %.2f ops/clk/SM\n", name, threads, ops / mx);
  }
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<0>("ex2.f32", 1);
  run<1>("cvt.bf16x2.f32", 1);
  run<2>("ex2.bf16x2 (pairs)", 1);
  run<3>("2ex2+cvt (elements)", 2);
  run<4>("ffma", 1);
  run<5>("cvt.bf16.f32", 1);
  run<6>("max3", 1);
  run<7>("cvt.f16x2.f32", 1);
  run<8>("ex2.f16x2 (pairs)", 1);
  return 0;
}
