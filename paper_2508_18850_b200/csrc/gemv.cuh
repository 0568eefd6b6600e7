// Row-tiled GEMV consumer shared by the attention (QKV), FFN and LM-head kernels.
//
// Weight layout ("row tiles"): rows are grouped in tiles of 4 consecutive
// rows stored chunk-major, [tile][chunk][4 rows][16 B], where a chunk is 16
// bytes of one row (8 fp16 or 4 fp32 weights).  A warp covers 8 chunks x 4
// rows per step: lane = 4*q + r reads chunk q+8k of row r, so the 32 lanes
// read 512 contiguous bytes (conflict-free LDS.128) and only 8 distinct
// activation chunks, which live in shared memory as fp32 in a lo/hi split
// layout (8 consecutive chunks = 128 contiguous bytes: one wavefront, no
// conversion).  Per 16-byte weight vector a lane issues one weight LDS, two
// activation LDS, the fp16->fp32 unpack and four packed FFMA2s; no per-row
// shuffles except a 3-step butterfly across the 8 chunk groups per tile.
//
// Activation layout for fp16 weights, row of C elements: element d at
//   (d%8 < 4 ? 0 : C/2) + (d/8)*4 + d%4        (lo half | hi half)
// and plain contiguous for fp32 weights.
#pragma once
#include <type_traits>

#include "stream.cuh"

namespace cfb {

constexpr int kTileRows = 4;

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
__device__ __forceinline__ unsigned long long u2_lo(const uint4& v) {
  return (static_cast<unsigned long long>(v.y) << 32) | v.x;
}
__device__ __forceinline__ unsigned long long u2_hi(const uint4& v) {
  return (static_cast<unsigned long long>(v.w) << 32) | v.z;
}

// position of activation element d in the smem layout of a C-long row
// (XH: activations kept as fp16 in smem, plain contiguous; used when the
// fp32 split layout does not fit, i.e. batch > 2 at Llama FFN widths)
template <typename T, bool XH = false>
__device__ __forceinline__ int xpos(int d, int C) {
  if constexpr (sizeof(T) == 2 && !XH) return ((d & 7) < 4 ? 0 : C / 2) + (d >> 3) * 4 + (d & 3);
  return d;
}
template <bool XH>
using XElem = typename std::conditional<XH, __half, float>::type;

// One tiles-mode item: for every tile in the item, the lanes' partial dot
// products of the tile's 4 rows (over the item's chunks) with B activation
// rows, reduced across the 8 chunk groups.  emit(row, sums) runs on all
// lanes; lanes 0..3 (chunk group 0) hold row (4*tile + lane)'s sums.
template <typename T, int QB, bool XH, class Emit>
__device__ __forceinline__ void tile_item(const Phase& P, const Item& it, const char* slot,
                                          const XElem<XH>* xs, int C, int B, int lane, Emit&& emit) {
  const int q = lane >> 2, r = lane & 3;
  const int nch = it.bytes / (it.nunits * 64);  // chunks per tile in this item
  const int ch0 = it.byte0 / 64;
  for (int t = 0; t < it.nunits; ++t) {
    const char* tile = slot + t * nch * 64;
    unsigned long long acc[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) acc[b] = 0ull;
#pragma unroll 4
    for (int c = q; c < nch; c += 8) {
      const uint4 wv = lds128(tile + (c * 4 + r) * 16);
      const int gc = ch0 + c;
      if constexpr (sizeof(T) == 2 && XH) {
        const __half2* h = reinterpret_cast<const __half2*>(&wv);
        const float2 w0 = __half22float2(h[0]), w1 = __half22float2(h[1]);
        const float2 w2 = __half22float2(h[2]), w3 = __half22float2(h[3]);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const uint4 xv = lds128(xs + (size_t)b * C + gc * 8);
            const __half2* xh = reinterpret_cast<const __half2*>(&xv);
            const float2 x0 = __half22float2(xh[0]), x1 = __half22float2(xh[1]);
            const float2 x2 = __half22float2(xh[2]), x3 = __half22float2(xh[3]);
            acc[b] = ffma2(f2_pack(w0.x, w0.y), f2_pack(x0.x, x0.y), acc[b]);
            acc[b] = ffma2(f2_pack(w1.x, w1.y), f2_pack(x1.x, x1.y), acc[b]);
            acc[b] = ffma2(f2_pack(w2.x, w2.y), f2_pack(x2.x, x2.y), acc[b]);
            acc[b] = ffma2(f2_pack(w3.x, w3.y), f2_pack(x3.x, x3.y), acc[b]);
          }
        }
      } else if constexpr (sizeof(T) == 2) {
        const __half2* h = reinterpret_cast<const __half2*>(&wv);
        const float2 w0 = __half22float2(h[0]), w1 = __half22float2(h[1]);
        const float2 w2 = __half22float2(h[2]), w3 = __half22float2(h[3]);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const float* xb = xs + (size_t)b * C;
            const uint4 lo = lds128(xb + gc * 4), hi = lds128(xb + C / 2 + gc * 4);
            acc[b] = ffma2(f2_pack(w0.x, w0.y), u2_lo(lo), acc[b]);
            acc[b] = ffma2(f2_pack(w1.x, w1.y), u2_hi(lo), acc[b]);
            acc[b] = ffma2(f2_pack(w2.x, w2.y), u2_lo(hi), acc[b]);
            acc[b] = ffma2(f2_pack(w3.x, w3.y), u2_hi(hi), acc[b]);
          }
        }
      } else {
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const uint4 xv = lds128(xs + (size_t)b * C + gc * 4);
            acc[b] = ffma2(u2_lo(wv), u2_lo(xv), acc[b]);
            acc[b] = ffma2(u2_hi(wv), u2_hi(xv), acc[b]);
          }
        }
      }
    }
    float s[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      float v = f2_sum(acc[b]);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      s[b] = v;
    }
    emit((it.unit0 + t) * kTileRows + r, s);
  }
}

// Tiles-mode GEMV phase with a deterministic cross-warp reduction: every
// warp adds its items' row partials into its private slice of `part`
// ([kNumConsumerWarps][B][rows]); finish(row, b, value) then runs for each
// (row < rows) with the warp slices summed in warp order.
template <typename T, int QB, bool XH = false, class Finish>
__device__ __forceinline__ void tiled_gemv_phase(const Phase& P, const Ring& ring, int warp,
                                                 int lane, int tid, int& cnt, const XElem<XH>* xs,
                                                 int C, int B, int rows, float* part,
                                                 Finish&& finish) {
  for (int i = tid; i < kNumConsumerWarps * B * rows; i += kConsumerThreads) part[i] = 0.f;
  consumer_sync();
  float* mine = part + (size_t)warp * B * rows;
  consume_phase(P, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    tile_item<T, QB, XH>(P, it, slot, xs, C, B, lane, [&](int row, const float (&s)[QB]) {
      if (lane < kTileRows && row < rows) {
#pragma unroll
        for (int b = 0; b < QB; ++b)
          if (b < B) mine[b * rows + row] += s[b];
      }
    });
  });
  consumer_sync();
  for (int i = tid; i < B * rows; i += kConsumerThreads) {
    float v = 0.f;
    for (int w = 0; w < kNumConsumerWarps; ++w) v += part[(size_t)w * B * rows + i];
    finish(i % rows, i / rows, v);
  }
}

// Residual-stream row loader: 4 consecutive fp32 values of row b starting at
// element 4*v.  The plain form reads resid; RMSNorm prologues take any loader.
struct ResidLoad {
  const float* resid;
  int D;
  __device__ __forceinline__ float4 operator()(int b, int v) const {
    return reinterpret_cast<const float4*>(resid + (size_t)b * D)[v];
  }
};

// x[b][d] = T((r[b][d] * (1/sqrt(mean_d(r^2) + eps))) * w[d]) as fp32 in the
// tile-GEMV activation layout (fp16 contiguous when XH), r[b] read through
// `ld` as float4s; `red` holds kNumConsumerWarps * B floats.  Each thread
// issues its (up to 4) independent 16-byte loads at once and keeps them in
// registers for the scaling pass, so the prologue costs ~one L2 round trip.
template <typename T, bool XH = false, class Load>
__device__ void rmsnorm_to_smem_ld(XElem<XH>* xs, Load&& ld, const T* w, int B, int D, float eps,
                                   float* red, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int nv = D / 4;
  constexpr int kReg = 4;
  for (int b = 0; b < B; ++b) {
    float4 c[kReg];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kReg; ++k) {
      const int v = tid + k * kConsumerThreads;
      c[k] = v < nv ? ld(b, v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < kReg; ++k)
      ss = fmaf(c[k].w, c[k].w, fmaf(c[k].z, c[k].z, fmaf(c[k].y, c[k].y, fmaf(c[k].x, c[k].x, ss))));
    for (int v = tid + kReg * kConsumerThreads; v < nv; v += kConsumerThreads) {
      const float4 a = ld(b, v);
      ss = fmaf(a.w, a.w, fmaf(a.z, a.z, fmaf(a.y, a.y, fmaf(a.x, a.x, ss))));
    }
    ss = warp_allsum(ss);
    if (lane == 0) red[b * kNumConsumerWarps + warp] = ss;
    consumer_sync();
    float tot = 0.f;
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) tot += red[b * kNumConsumerWarps + w2];
    const float inv = 1.0f / sqrtf(__fdiv_rn(tot, (float)D) + eps);
    auto emit = [&](const float4& a, int v) {
      float g[4];
      if constexpr (sizeof(T) == 2) {
        const uint2 wv = *reinterpret_cast<const uint2*>(w + 4 * v);
        const float2 g01 = __half22float2(*reinterpret_cast<const __half2*>(&wv.x));
        const float2 g23 = __half22float2(*reinterpret_cast<const __half2*>(&wv.y));
        g[0] = g01.x; g[1] = g01.y; g[2] = g23.x; g[3] = g23.y;
      } else {
        const float4 wv = *reinterpret_cast<const float4*>(w + 4 * v);
        g[0] = wv.x; g[1] = wv.y; g[2] = wv.z; g[3] = wv.w;
      }
      float o[4] = {__fmul_rn(__fmul_rn(a.x, inv), g[0]), __fmul_rn(__fmul_rn(a.y, inv), g[1]),
                    __fmul_rn(__fmul_rn(a.z, inv), g[2]), __fmul_rn(__fmul_rn(a.w, inv), g[3])};
      if constexpr (XH) {
        __half2* dst = reinterpret_cast<__half2*>(xs + (size_t)b * D + 4 * v);
        dst[0] = __floats2half2_rn(o[0], o[1]);
        dst[1] = __floats2half2_rn(o[2], o[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = round_to<T>(o[e]);
        // 4 consecutive elements stay contiguous in both activation layouts
        *reinterpret_cast<float4*>(xs + (size_t)b * D + xpos<T>(4 * v, D)) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
    };
#pragma unroll
    for (int k = 0; k < kReg; ++k)
      if (tid + k * kConsumerThreads < nv) emit(c[k], tid + k * kConsumerThreads);
    for (int v = tid + kReg * kConsumerThreads; v < nv; v += kConsumerThreads) emit(ld(b, v), v);
  }
  consumer_sync();
}

template <typename T, bool XH = false>
__device__ __forceinline__ void rmsnorm_to_smem(XElem<XH>* xs, const float* resid, const T* w, int B,
                                                int D, float eps, float* red, int tid) {
  rmsnorm_to_smem_ld<T, XH>(xs, ResidLoad{resid, D}, w, B, D, eps, red, tid);
}

// n_rows rows of C T-activations (16-byte aligned) from global memory into
// the fp32 tile-GEMV layout.
template <typename T, bool XH = false>
__device__ __forceinline__ void load_act_to_smem(XElem<XH>* xs, const T* x, int n_rows, int C,
                                                 int tid) {
  constexpr int epv = Elem<T>::kPerVec;
  const uint4* s = reinterpret_cast<const uint4*>(x);
  const int vpr = C / epv;
  if constexpr (XH) {  // fp16 -> fp16, contiguous
    uint4* d = reinterpret_cast<uint4*>(xs);
    for (int v = tid; v < n_rows * vpr; v += kConsumerThreads) d[v] = __ldcg(s + v);
  } else {
    for (int v = tid; v < n_rows * vpr; v += kConsumerThreads) {
      const int b = v / vpr, k = v % vpr;
      float f[epv];
      Elem<T>::unpack(__ldcg(s + v), f);
      float* xb = xs + (size_t)b * C;
      if constexpr (epv == 8) {
        *reinterpret_cast<float4*>(xb + k * 4) = make_float4(f[0], f[1], f[2], f[3]);
        *reinterpret_cast<float4*>(xb + C / 2 + k * 4) = make_float4(f[4], f[5], f[6], f[7]);
      } else {
        *reinterpret_cast<float4*>(xb + k * 4) = make_float4(f[0], f[1], f[2], f[3]);
      }
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
