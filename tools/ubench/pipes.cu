// Issue-throughput microbenchmark of the FMA flavours the GEMV consumers use
// (sm_100a): FFMA, FFMA2, FHFMA (fma.rn.f32.f16) and HADD2.F32 conversion.
// One CTA of `warps` warps per SM, 8 independent accumulator chains/thread.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float fhfma(unsigned a, unsigned b, float c) {
  float d;
  asm volatile("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
               "fma.rn.f32.f16 %0, al, bl, %3;\n\t}" : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters, unsigned seed) {
  float acc[8];
  unsigned long long acc2[8];
  for (int i = 0; i < 8; ++i) { acc[i] = 0.f; acc2[i] = 0ull; }
  unsigned a = seed ^ threadIdx.x, b = seed * 7 + threadIdx.x;
  float fa = __uint_as_float(a & 0x3f7fffff), fb = __uint_as_float(b & 0x3f7fffff);
  unsigned long long pa = ((unsigned long long)a << 32) | b, pb = pa ^ 0x1234;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) acc[i] = fmaf(fa, fb, acc[i]);
      if (MODE == 1) acc2[i] = ffma2(pa, pb, acc2[i]);
      if (MODE == 2) acc[i] = fhfma(a + i, b, acc[i]);
      if (MODE == 3) acc[i] += __half2float(__ushort_as_half((unsigned short)(a + i + it)));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += acc[i] + __uint_as_float((unsigned)acc2[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"FFMA", "FFMA2", "FHFMA", "HADD2.F32+FADD"};
  for (int warps : {2, 8, 16}) {
    for (int m = 0; m < 4; ++m) {
      const int iters = 4096;
      auto f = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
      f<<<148, warps * 32>>>(out, cyc, iters, 1);
      f<<<148, warps * 32>>>(out, cyc, iters, 1);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = (double)iters * 8 * warps;  // warp-instructions per SM
      printf("warps=%2d %-16s cycles %8lld  warp-instr/cycle/SM %.2f\n", warps, names[m], c, instr / c);
    }
  }
  return 0;
}
