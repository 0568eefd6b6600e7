// Row-GEMV consumer shared by the attention, FFN and LM-head kernels:
// dot products of streamed weight rows (K-major, in a ring slot) with B
// activation rows held in shared memory.  Lanes stride over 16-byte vectors
// of a row; a row that spans several slot pieces keeps its partial sums in
// registers until its last piece, then a warp butterfly finishes the sum.
#pragma once
#include "stream.cuh"

namespace cfb {

__device__ __forceinline__ float warp_allsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned long long f2_pack(float x, float y) {
  return (static_cast<unsigned long long>(__float_as_uint(y)) << 32) | __float_as_uint(x);
}
// c += a * b on packed fp32 pairs (sm_100 FFMA2)
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float f2_sum(unsigned long long v) {
  return __uint_as_float(static_cast<unsigned>(v)) + __uint_as_float(static_cast<unsigned>(v >> 32));
}

// Load 8 activations (elements [k, k+8) of an XT row in smem) as 4 fp32 pairs.
template <typename XT>
__device__ __forceinline__ void load_x8(const XT* x, unsigned long long (&xp)[4]) {
  if constexpr (sizeof(XT) == 4) {
    const uint4 a = lds128(x), b = lds128(x + 4);
    xp[0] = (static_cast<unsigned long long>(a.y) << 32) | a.x;
    xp[1] = (static_cast<unsigned long long>(a.w) << 32) | a.z;
    xp[2] = (static_cast<unsigned long long>(b.y) << 32) | b.x;
    xp[3] = (static_cast<unsigned long long>(b.w) << 32) | b.z;
  } else {
    float f[8];
    Elem<XT>::unpack(lds128(x), f);
#pragma unroll
    for (int i = 0; i < 4; ++i) xp[i] = f2_pack(f[2 * i], f[2 * i + 1]);
  }
}

// Weights T (fp16 or fp32) streamed in slots; activations XT (fp32 or T) in
// smem rows of stride `xstride`.  Per 16-byte weight vector: one LDS.128,
// the fp16->fp32 unpack, and packed FFMA2s into two interleaved partial sums.
template <typename T, typename XT, int QB>
struct RowDot {
  unsigned long long acc[QB];

  // done(row_index, sums) runs on all lanes with warp-reduced sums[QB].
  template <class Done>
  __device__ __forceinline__ void item(const Phase& P, const Item& it, const char* slot,
                                       const XT* xs, int xstride, int B, int lane, Done&& done) {
    constexpr int epv = Elem<T>::kPerVec;
    const int row_b = (P.pieces == 1) ? P.row_bytes : it.bytes;
    const int col0 = it.byte0 / static_cast<int>(sizeof(T));
    for (int rr = 0; rr < it.nrows; ++rr) {
      const char* row = slot + rr * row_b;
      if (it.piece == 0) {
#pragma unroll
        for (int b = 0; b < QB; ++b) acc[b] = 0ull;
      }
      const int nvec = row_b / 16;
#pragma unroll 4
      for (int v = lane; v < nvec; v += 32) {
        float w[epv];
        Elem<T>::unpack(lds128(row + 16 * v), w);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const XT* xb = xs + (size_t)b * xstride + col0 + v * epv;
#pragma unroll
            for (int h8 = 0; h8 < epv / 8 + (epv < 8 ? 1 : 0); ++h8) {
              if constexpr (epv >= 8) {
                unsigned long long xp[4];
                load_x8<XT>(xb + 8 * h8, xp);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                  acc[b] = ffma2(f2_pack(w[8 * h8 + 2 * i], w[8 * h8 + 2 * i + 1]), xp[i], acc[b]);
              } else {  // fp32 weights: 4 per vector
                float xv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) xv[i] = Elem<XT>::to_f(xb[i]);
                acc[b] = ffma2(f2_pack(w[0], w[1]), f2_pack(xv[0], xv[1]), acc[b]);
                acc[b] = ffma2(f2_pack(w[2], w[3]), f2_pack(xv[2], xv[3]), acc[b]);
              }
            }
          }
        }
      }
      if (it.piece == P.pieces - 1) {
        float s[QB];
#pragma unroll
        for (int b = 0; b < QB; ++b) s[b] = (b < B) ? warp_allsum(f2_sum(acc[b])) : 0.f;
        done(it.row0 + rr, s);
      }
    }
  }
};

// x[b][d] = T((resid[b][d] * (1/sqrt(mean_d(resid^2) + eps))) * w[d]) for all
// consumer threads, stored as XT (the fp16-rounded value, widened when XT is
// float); `red` holds kNumConsumerWarps * B floats.
template <typename T, typename XT>
__device__ void rmsnorm_to_smem(XT* xs, const float* resid, const T* w, int B, int D, float eps,
                                float* red, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int b = 0; b < B; ++b) {
    float ss = 0.f;
    for (int d = tid; d < D; d += kConsumerThreads) {
      const float v = resid[(size_t)b * D + d];
      ss = fmaf(v, v, ss);
    }
    ss = warp_allsum(ss);
    if (lane == 0) red[b * kNumConsumerWarps + warp] = ss;
  }
  consumer_sync();
  for (int b = 0; b < B; ++b) {
    float tot = 0.f;
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) tot += red[b * kNumConsumerWarps + w2];
    const float inv = 1.0f / sqrtf(__fdiv_rn(tot, (float)D) + eps);
    for (int d = tid; d < D; d += kConsumerThreads) {
      const float v = __fmul_rn(__fmul_rn(resid[(size_t)b * D + d], inv), Elem<T>::to_f(w[d]));
      xs[(size_t)b * D + d] = static_cast<XT>(round_to<T>(v));
    }
  }
  consumer_sync();
}

// Copy n T activations (16-byte aligned) from global into shared memory as XT.
template <typename T, typename XT>
__device__ __forceinline__ void copy_to_smem(XT* xs, const T* x, int n_elems, int tid) {
  if constexpr (sizeof(T) == sizeof(XT)) {
    const uint4* s = reinterpret_cast<const uint4*>(x);
    uint4* d = reinterpret_cast<uint4*>(xs);
    for (int v = tid; v < n_elems * (int)sizeof(T) / 16; v += kConsumerThreads) d[v] = __ldcg(s + v);
  } else {
    constexpr int epv = Elem<T>::kPerVec;
    const uint4* s = reinterpret_cast<const uint4*>(x);
    for (int v = tid; v < n_elems / epv; v += kConsumerThreads) {
      float f[epv];
      Elem<T>::unpack(__ldcg(s + v), f);
#pragma unroll
      for (int e = 0; e < epv; ++e) xs[v * epv + e] = f[e];
    }
  }
  consumer_sync();
}

// Grid-wide barrier among the consumer warps of all CTAs (grid <= #SMs,
// one CTA per SM, so every CTA is resident).  Monotonic 64-bit counter: the
// n-th use waits for n * gridDim.x arrivals, so it never needs resetting.
__device__ __forceinline__ void grid_barrier(unsigned long long* counter, int tid) {
  __threadfence();
  consumer_sync();
  if (tid == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomicAdd(counter, 1ull);
    const unsigned long long target = (old / g + 1) * g;
    while (ld_acquire_u64(counter) < target) __nanosleep(64);
  }
  consumer_sync();
}

}  // namespace cfb
