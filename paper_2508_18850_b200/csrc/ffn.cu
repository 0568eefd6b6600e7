// Fused SwiGLU FFN decode kernel (one launch): [RMSNorm ->] gate/up GEMV ->
// SiLU(gate) * up -> down GEMV [-> + residual].
//
// Reference semantics: ffn_reference(z, w1, w2, w3, "silu")
// (pkg/src/clusterdec/oracle.py:112-131) = (silu(z w1^T) * (z w2^T)) w3^T.
// The reference has no fused counterpart; this kernel is the
// north-star "gate/up GEMV, SiLU*mul and down GEMV in one launch".
//
// Persistent grid of one CTA per SM.  CTA i owns intermediate rows
// [i*F/G, (i+1)*F/G) (gate and up interleaved: packed row 2f = w1[f],
// 2f+1 = w2[f]) and output rows [i*D/G, (i+1)*D/G) of w3.  The activation
// vector crosses CTAs once, through global memory and a grid barrier; the
// producer warp keeps streaming this CTA's w3 rows into the ring while the
// barrier is pending, so HBM never idles at the phase boundary.
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct FfnParams {
  int B, D, F, flags, spw;
  float eps;
  const void* x;          // [B][D] T (no CFB_NORM)
  const float* resid;     // [B][D] fp32
  const void* norm_w;     // [D] T
  const void* w_gu;       // [F][2][D] T
  const void* w_dn;       // [D][F] T
  void* act;              // [B][F] T workspace
  float* out;             // [B][D] fp32
  unsigned long long* barrier;
};

// x (phase 0 input, B x D) and act (phase 1 input, B x F) are never live at
// the same time and share one region.
struct FfnLayout {
  int bars, x, gu, act, red, total;
};

__host__ __device__ inline FfnLayout ffn_layout(int B, int D, int F, int G, int tb, int spw) {
  FfnLayout L;
  const int fmax = F / G + 1;
  const int xb = B * D * tb, ab = B * F * tb;
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.x = o;
  L.act = o;   o += (((xb > ab) ? xb : ab) + 15) & ~15;
  L.gu = o;    o += (2 * B * fmax * 4 + 15) & ~15;
  L.red = o;   o += (kNumConsumerWarps * B * 4 + 15) & ~15;
  L.total = o;
  return L;
}

template <typename T, int QB>
__global__ void __launch_bounds__(kThreads, 1) ffn_swiglu_kernel(const FfnParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  const int B = p.B, D = p.D, F = p.F, G = gridDim.x, i = blockIdx.x;
  const FfnLayout L = ffn_layout(B, D, F, G, tb, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int f0 = (int)((long long)i * F / G), f1 = (int)((long long)(i + 1) * F / G);
  const int c0 = (int)((long long)i * D / G), c1 = (int)((long long)(i + 1) * D / G);
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const Phase P0 = make_phase(static_cast<const T*>(p.w_gu) + (size_t)2 * f0 * D, nullptr,
                              2 * (f1 - f0), D * tb);
  const Phase P1 = make_phase(static_cast<const T*>(p.w_dn) + (size_t)c0 * F, nullptr, c1 - c0,
                              F * tb);
  if (warp == kNumConsumerWarps) {
    const Phase ph[2] = {P0, P1};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  T* xs = reinterpret_cast<T*>(smem + L.x);
  float* gu = reinterpret_cast<float*>(smem + L.gu);  // [B][2*(f1-f0)]
  T* acts = reinterpret_cast<T*>(smem + L.act);
  float* red = reinterpret_cast<float*>(smem + L.red);
  const int nloc = 2 * (f1 - f0);

  if (p.flags & CFB_NORM)
    rmsnorm_to_smem<T, T>(xs, p.resid, static_cast<const T*>(p.norm_w), B, D, p.eps, red, tid);
  else
    copy_to_smem<T, T>(xs, static_cast<const T*>(p.x), B * D, tid);

  int cnt = 0;
  RowDot<T, T, QB> rd;
  consume_phase(P0, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    rd.item(P0, it, slot, xs, D, B, lane, [&](int row, const float (&s)[QB]) {
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < QB; ++b)
          if (b < B) gu[b * nloc + row] = s[b];
      }
    });
  });
  consumer_sync();
  T* act_g = static_cast<T*>(p.act);
  for (int idx = tid; idx < B * (f1 - f0); idx += kConsumerThreads) {
    const int b = idx / (f1 - f0), j = idx % (f1 - f0);
    const float g = gu[b * nloc + 2 * j], u = gu[b * nloc + 2 * j + 1];
    const float sl = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
    act_g[(size_t)b * F + f0 + j] = Elem<T>::from_f(__fmul_rn(sl, u));
  }
  grid_barrier(p.barrier, tid);
  copy_to_smem<T, T>(acts, act_g, B * F, tid);

  RowDot<T, T, QB> rd1;
  consume_phase(P1, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    rd1.item(P1, it, slot, acts, F, B, lane, [&](int row, const float (&s)[QB]) {
      if (lane == 0) {
        const int c = c0 + row;
#pragma unroll
        for (int b = 0; b < QB; ++b)
          if (b < B) {
            const float r = (p.flags & CFB_RESID) ? p.resid[(size_t)b * D + c] : 0.f;
            p.out[(size_t)b * D + c] = (p.flags & CFB_RESID) ? __fadd_rn(r, s[b]) : s[b];
          }
      }
    });
  });
}

template <typename T, int QB>
static int launch_ffn_inst(const FfnParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = ffn_swiglu_kernel<T, QB>;
  static bool configured = false;
  if (!configured) {
    CFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    configured = true;
  }
  kern<<<grid, kThreads, smem, st>>>(p);
  CFB_CUDA(cudaGetLastError());
  return CFB_OK;
}

int ffn_decode(const cfb_ffn_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  const int tb = a->dtype;
  if (tb != CFB_F16 && tb != CFB_F32) return set_error(CFB_ERR_ARGUMENT, "bad dtype");
  if (a->batch < 1 || a->batch > 8) return set_error(CFB_ERR_DIMENSION, "ffn batch must be in [1, 8]");
  if ((a->hidden * tb) % 16 || (a->inter * tb) % 16)
    return set_error(CFB_ERR_DIMENSION, "hidden and inter must give 16-byte rows");
  if (!a->w_gu || !a->w_dn || !a->act || !a->out || !a->barrier)
    return set_error(CFB_ERR_ARGUMENT, "null weight / workspace pointer");
  if ((a->flags & CFB_NORM) ? (!a->resid || !a->norm_w) : !a->x)
    return set_error(CFB_ERR_ARGUMENT, "missing activation input");
  if ((a->flags & CFB_RESID) && !a->resid) return set_error(CFB_ERR_ARGUMENT, "CFB_RESID needs resid");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = a->grid > 0 ? a->grid : sms;
  grid = grid > sms ? sms : grid;  // grid barrier: every CTA must be co-resident
  if (grid > a->inter) grid = a->inter;
  int spw = tuned_spw();
  FfnLayout L = ffn_layout(a->batch, a->hidden, a->inter, grid, tb, spw);
  while (L.total > kMaxSmem && spw > 1) L = ffn_layout(a->batch, a->hidden, a->inter, grid, tb, --spw);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "ffn schedule needs %d B of shared memory (max %d)", L.total,
                     kMaxSmem);
  FfnParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.F = a->inter;
  p.flags = a->flags;
  p.spw = spw;
  p.eps = a->eps;
  p.x = a->x;
  p.resid = a->resid;
  p.norm_w = a->norm_w;
  p.w_gu = a->w_gu;
  p.w_dn = a->w_dn;
  p.act = a->act;
  p.out = a->out;
  p.barrier = a->barrier;
  const size_t smem = L.total;
  if (tb == 2) {
    if (p.B == 1) return launch_ffn_inst<__half, 1>(p, grid, smem, st);
    if (p.B == 2) return launch_ffn_inst<__half, 2>(p, grid, smem, st);
    if (p.B <= 4) return launch_ffn_inst<__half, 4>(p, grid, smem, st);
    return launch_ffn_inst<__half, 8>(p, grid, smem, st);
  }
  if (p.B == 1) return launch_ffn_inst<float, 1>(p, grid, smem, st);
  if (p.B <= 4) return launch_ffn_inst<float, 4>(p, grid, smem, st);
  return launch_ffn_inst<float, 8>(p, grid, smem, st);
}

}  // namespace cfb
