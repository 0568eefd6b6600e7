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

template <typename T, int QB>
struct RowDot {
  float acc[QB];

  // done(row_index, sums) runs on all lanes with warp-reduced sums[QB].
  template <class Done>
  __device__ __forceinline__ void item(const Phase& P, const Item& it, const char* slot,
                                       const T* xs, int xstride, int B, int lane, Done&& done) {
    constexpr int epv = Elem<T>::kPerVec;
    const int row_b = (P.pieces == 1) ? P.row_bytes : it.bytes;
    const int col0 = it.byte0 / static_cast<int>(sizeof(T));
    for (int rr = 0; rr < it.nrows; ++rr) {
      const char* row = slot + rr * row_b;
      if (it.piece == 0) {
#pragma unroll
        for (int b = 0; b < QB; ++b) acc[b] = 0.f;
      }
      const int nvec = row_b / 16;
#pragma unroll 4
      for (int v = lane; v < nvec; v += 32) {
        float w[epv];
        Elem<T>::unpack(lds128(row + 16 * v), w);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            float xv[epv];
            Elem<T>::unpack(lds128(xs + (size_t)b * xstride + col0 + v * epv), xv);
#pragma unroll
            for (int e = 0; e < epv; ++e) acc[b] = fmaf(w[e], xv[e], acc[b]);
          }
        }
      }
      if (it.piece == P.pieces - 1) {
        float s[QB];
#pragma unroll
        for (int b = 0; b < QB; ++b) s[b] = (b < B) ? warp_allsum(acc[b]) : 0.f;
        done(it.row0 + rr, s);
      }
    }
  }
};

// x[b][d] = T((resid[b][d] * (1/sqrt(mean_d(resid^2) + eps))) * w[d]) for all
// consumer threads; `red` holds kNumConsumerWarps * B floats.
template <typename T>
__device__ void rmsnorm_to_smem(T* xs, const float* resid, const T* w, int B, int D, float eps,
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
      xs[(size_t)b * D + d] = Elem<T>::from_f(v);
    }
  }
  consumer_sync();
}

// Copy B*D T activations (16-byte rows) from global into shared memory.
template <typename T>
__device__ __forceinline__ void copy_to_smem(T* xs, const T* x, int n_elems, int tid) {
  const uint4* s = reinterpret_cast<const uint4*>(x);
  uint4* d = reinterpret_cast<uint4*>(xs);
  for (int v = tid; v < n_elems * (int)sizeof(T) / 16; v += kConsumerThreads) d[v] = __ldcg(s + v);
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
