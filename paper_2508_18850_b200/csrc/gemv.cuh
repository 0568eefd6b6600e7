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
// d = float(lo/hi half of a) * float(lo/hi half of b) + c   (sm_100 FHFMA)
__device__ __forceinline__ float fma_f16_lo(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.f16 %0, al, bl, %3;\n\t}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fma_f16_hi(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.f16 %0, ah, bh, %3;\n\t}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
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
// Multiply-accumulate of one 16-byte weight chunk (global chunk index gc)
// with the B activation rows.
template <typename T, int QB, bool XH>
__device__ __forceinline__ void chunk_mac(unsigned long long (&acc)[QB], const uint4& wv, int gc,
                                          const XElem<XH>* xs, int C, int B) {
  if constexpr (sizeof(T) == 2 && XH) {
    // fp16 weights x fp16 activations, fp32 accumulate: one FHFMA per weight
    // (fma.rn.f32.f16 - the f16 x f16 product is exact in fp32, so this is
    // bit-identical to converting both operands first), no conversions
    const uint32_t wr[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      if (b < B) {
        const uint4 xv = lds128(xs + (size_t)b * C + gc * 8);
        const uint32_t xr[4] = {xv.x, xv.y, xv.z, xv.w};
        float lo = __uint_as_float(static_cast<uint32_t>(acc[b]));
        float hi = __uint_as_float(static_cast<uint32_t>(acc[b] >> 32));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          lo = fma_f16_lo(wr[j], xr[j], lo);
          hi = fma_f16_hi(wr[j], xr[j], hi);
        }
        acc[b] = f2_pack(lo, hi);
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

// One tiles-mode item: for every tile in the item, the lanes' partial dot
// products of the tile's 4 rows (over the item's chunks) with B activation
// rows, reduced across the 8 chunk groups.  emit(row, sums) runs on all
// lanes; lanes 0..3 (chunk group 0) hold row (4*tile + lane)'s sums.  Short
// rows (K = head_dim in the O-projection: 2 chunks per lane per tile) are
// processed TG tiles at a time so the butterflies of TG tiles interleave
// instead of serialising on shuffle latency.
template <typename T, int QB, bool XH, class Emit>
__device__ __forceinline__ void tile_item(const Phase& P, const Item& it, const char* slot,
                                          const XElem<XH>* xs, int C, int B, int lane, Emit&& emit) {
  constexpr int TG = QB == 1 ? 8 : (QB <= 2 ? 4 : (QB <= 4 ? 2 : 1));
  const int q = lane >> 2, r = lane & 3;
  const int nch = it.bytes / (it.nunits * 64);  // chunks per tile in this item
  const int ch0 = it.byte0 / 64;
  if (TG > 1 && nch <= 16) {
    // short rows: TG tiles per group, at most 2 chunks per lane per tile
    for (int t0 = 0; t0 < it.nunits; t0 += TG) {
      unsigned long long acc[TG][QB];
#pragma unroll
      for (int u = 0; u < TG; ++u)
#pragma unroll
        for (int b = 0; b < QB; ++b) acc[u][b] = 0ull;
      if (t0 + TG <= it.nunits) {  // full group: straight-line, loads hoisted
        uint4 wv[TG][2];
#pragma unroll
        for (int u = 0; u < TG; ++u)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            wv[u][k] = (q + 8 * k < nch) ? lds128(slot + (((t0 + u) * nch + q + 8 * k) * 4 + r) * 16)
                                         : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < TG; ++u)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (q + 8 * k < nch) chunk_mac<T, QB, XH>(acc[u], wv[u][k], ch0 + q + 8 * k, xs, C, B);
      } else {
#pragma unroll
        for (int u = 0; u < TG; ++u) {
          if (t0 + u < it.nunits) {
            const char* tile = slot + (t0 + u) * nch * 64;
#pragma unroll
            for (int k = 0; k < 2; ++k)
              if (q + 8 * k < nch)
                chunk_mac<T, QB, XH>(acc[u], lds128(tile + ((q + 8 * k) * 4 + r) * 16),
                                     ch0 + q + 8 * k, xs, C, B);
          }
        }
      }
      float s[TG][QB];
#pragma unroll
      for (int u = 0; u < TG; ++u)
#pragma unroll
        for (int b = 0; b < QB; ++b) s[u][b] = f2_sum(acc[u][b]);
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1)
#pragma unroll
        for (int u = 0; u < TG; ++u)
#pragma unroll
          for (int b = 0; b < QB; ++b) s[u][b] += __shfl_xor_sync(0xffffffffu, s[u][b], o);
#pragma unroll
      for (int u = 0; u < TG; ++u)
        if (t0 + u < it.nunits) emit((it.unit0 + t0 + u) * kTileRows + r, s[u]);
    }
    return;
  }
  for (int t = 0; t < it.nunits; ++t) {
    const char* tile = slot + t * nch * 64;
    unsigned long long acc[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) acc[b] = 0ull;
#pragma unroll 4
    for (int c = q; c < nch; c += 8)
      chunk_mac<T, QB, XH>(acc, lds128(tile + (c * 4 + r) * 16), ch0 + c, xs, C, B);
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

// Short-row GEMV item (rows mode, K = C elements, C*sizeof(T) small: the
// O-projection's K = head_dim): one lane per row (L lanes per row when a row
// exceeds 16 chunks), so there are no cross-lane reductions at all.  Rows are
// stored chunk-rotated - logical chunk k of slice row g sits at physical chunk
// (k + g) mod nch - so the 32 lanes of a warp, each reading "its" row, hit all
// eight 16-byte bank groups (conflict-free LDS.128).  The activation chunk is
// the same for every lane (broadcast).  emit(g, sums) runs on the row's lane 0.
template <typename T, int QB, int NCH, class Emit>
__device__ __forceinline__ void rowlane_item_fixed(const Item& it, const char* slot, const T* a,
                                                   int B, int lane, Emit&& emit) {
  // NCH chunks per row, one lane per row, no runtime conditions in the row body
  constexpr int tb = sizeof(T), epc = 16 / tb, C = NCH * epc, rb = C * tb;
  for (int r0 = 0; r0 < it.nunits; r0 += 32) {
    const int row = r0 + lane;
    const bool valid = row < it.nunits;
    const int g = it.unit0 + row;
    const char* rp = slot + (size_t)(valid ? row : 0) * rb;
    uint4 wv[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) wv[k] = lds128(rp + ((k + g) & (NCH - 1)) * 16);
    float s[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (b < B) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const uint4 av = lds128(a + (size_t)b * C + k * epc);
          if constexpr (tb == 2) {
            acc[0] = fma_f16_lo(wv[k].x, av.x, acc[0]);
            acc[1] = fma_f16_hi(wv[k].x, av.x, acc[1]);
            acc[2] = fma_f16_lo(wv[k].y, av.y, acc[2]);
            acc[3] = fma_f16_hi(wv[k].y, av.y, acc[3]);
            acc[0] = fma_f16_lo(wv[k].z, av.z, acc[0]);
            acc[1] = fma_f16_hi(wv[k].z, av.z, acc[1]);
            acc[2] = fma_f16_lo(wv[k].w, av.w, acc[2]);
            acc[3] = fma_f16_hi(wv[k].w, av.w, acc[3]);
          } else {
            acc[0] = fmaf(__uint_as_float(wv[k].x), __uint_as_float(av.x), acc[0]);
            acc[1] = fmaf(__uint_as_float(wv[k].y), __uint_as_float(av.y), acc[1]);
            acc[2] = fmaf(__uint_as_float(wv[k].z), __uint_as_float(av.z), acc[2]);
            acc[3] = fmaf(__uint_as_float(wv[k].w), __uint_as_float(av.w), acc[3]);
          }
        }
      }
      s[b] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
    if (valid) emit(g, s);
  }
}

template <typename T, int QB, class Emit>
__device__ __forceinline__ void rowlane_item(const Item& it, const char* slot, const T* a, int C,
                                             int B, int lane, Emit&& emit) {
  constexpr int tb = sizeof(T);
  constexpr int epc = 16 / tb;
  constexpr int kMaxChunks = 16;  // chunks per lane
  const int nch = C * tb / 16, rb = C * tb;
  if (nch == 16) return rowlane_item_fixed<T, QB, 16>(it, slot, a, B, lane, emit);
  if (nch == 8) return rowlane_item_fixed<T, QB, 8>(it, slot, a, B, lane, emit);
  const int L = nch > kMaxChunks ? nch / kMaxChunks : 1;
  const int sub = lane % L, lr = lane / L, step = 32 / L;
  for (int r0 = 0; r0 < it.nunits; r0 += step) {
    const int row = r0 + lr;
    const bool valid = row < it.nunits;
    const int g = it.unit0 + row;
    const char* rp = slot + (size_t)(valid ? row : 0) * rb;
    float acc[QB][2];
#pragma unroll
    for (int b = 0; b < QB; ++b) acc[b][0] = acc[b][1] = 0.f;
    uint4 wv[kMaxChunks];
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int k = sub + L * i;
      if (k < nch) wv[i] = lds128(rp + ((k + g) & (nch - 1)) * 16);
    }
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int k = sub + L * i;
      if (k < nch) {
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const uint4 av = lds128(a + (size_t)b * C + k * epc);
            if constexpr (tb == 2) {
              const uint32_t wr[4] = {wv[i].x, wv[i].y, wv[i].z, wv[i].w};
              const uint32_t ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc[b][0] = fma_f16_lo(wr[j], ar[j], acc[b][0]);
                acc[b][1] = fma_f16_hi(wr[j], ar[j], acc[b][1]);
              }
            } else {
              acc[b][0] = fmaf(__uint_as_float(wv[i].x), __uint_as_float(av.x), acc[b][0]);
              acc[b][1] = fmaf(__uint_as_float(wv[i].y), __uint_as_float(av.y), acc[b][1]);
              acc[b][0] = fmaf(__uint_as_float(wv[i].z), __uint_as_float(av.z), acc[b][0]);
              acc[b][1] = fmaf(__uint_as_float(wv[i].w), __uint_as_float(av.w), acc[b][1]);
            }
          }
        }
      }
    }
    float s[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      s[b] = acc[b][0] + acc[b][1];
      for (int o = 1; o < L; o <<= 1) s[b] += __shfl_xor_sync(0xffffffffu, s[b], o);
    }
    if (valid && sub == 0) emit(g, s);
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
  // the gains do not depend on the reduction: load them with the first batch
  // (one round trip instead of two - the gain rows are usually cold in L2)
  using GVec = typename std::conditional<sizeof(T) == 2, uint2, float4>::type;
  GVec gv[kReg];
#pragma unroll
  for (int k = 0; k < kReg; ++k) {
    const int v = tid + k * kConsumerThreads;
    if (v < nv) gv[k] = *reinterpret_cast<const GVec*>(w + 4 * v);
  }
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
    auto emit = [&](const float4& a, int v, const GVec* pre) {
      float g[4];
      if constexpr (sizeof(T) == 2) {
        const uint2 wv = pre ? *pre : *reinterpret_cast<const uint2*>(w + 4 * v);
        const float2 g01 = __half22float2(*reinterpret_cast<const __half2*>(&wv.x));
        const float2 g23 = __half22float2(*reinterpret_cast<const __half2*>(&wv.y));
        g[0] = g01.x; g[1] = g01.y; g[2] = g23.x; g[3] = g23.y;
      } else {
        const float4 wv = pre ? *pre : *reinterpret_cast<const float4*>(w + 4 * v);
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
      if (tid + k * kConsumerThreads < nv) emit(c[k], tid + k * kConsumerThreads, &gv[k]);
    for (int v = tid + kReg * kConsumerThreads; v < nv; v += kConsumerThreads) emit(ld(b, v), v, nullptr);
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
  consumer_sync();
  if (tid == 0) {
    __threadfence();  // cumulative over the CTA's writes ordered by the bar.sync above
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomicAdd(counter, 1ull);
    const unsigned long long target = (old / g + 1) * g;
    while (ld_acquire_u64(counter) < target) __nanosleep(64);
  }
  consumer_sync();
}

}  // namespace cfb
