// Final RMSNorm + LM-head GEMV + greedy argmax (one launch), and the
// token-embedding gather that starts a decode step.  No reference
// counterpart (SPEC.md:298 lists the LM head as a non-goal); these close the
// north-star decode loop around the fused attention / FFN modules.
//
// Argmax semantics = numpy.argmax: first index of the maximum.  Each CTA
// reduces its vocabulary slice; the last CTA to finish (ticket) reduces the
// per-CTA candidates in CTA order, writes the token and advances the step
// position, so a captured CUDA graph can be replayed step after step.
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct LmParams {
  int B, D, V, flags, spw, sleep_max;
  float eps;
  const float* resid;
  const void* norm_w;
  const void* w;        // [V][D] T
  float* logits;        // [B][V] fp32 (nullable)
  float* cand_val;      // [G][B]
  int* cand_idx;        // [G][B]
  unsigned* ticket;     // 1 counter
  int* token_out;       // [B]
  int* step_pos;        // advanced by 1 when non-null
};

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi) || (bv != bv);  // NaN-free inputs assumed
}

template <typename T, int QB>
__global__ void __launch_bounds__(kThreads, 1) lm_head_kernel(const LmParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  const int B = p.B, D = p.D, V = p.V, G = gridDim.x, i = blockIdx.x;
  const int TV = (V + kTileRows - 1) / kTileRows;
  const int t0 = (int)((long long)i * TV / G), t1 = (int)((long long)(i + 1) * TV / G);
  const int rows = kTileRows * (t1 - t0);
  const int rows_max = kTileRows * ((TV + G - 1) / G);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes(p.spw));
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  constexpr bool XH = sizeof(T) == 2;  // fp16 activations (FHFMA GEMV path)
  XElem<XH>* xs = reinterpret_cast<XElem<XH>*>(smem + ring_bytes(p.spw) + 2 * kNumSlots * 8);
  float* part = reinterpret_cast<float*>(smem + ring_bytes(p.spw) + 2 * kNumSlots * 8) + B * D;
  float* red = part + kNumConsumerWarps * B * rows_max;
  float* wv = red + kNumConsumerWarps * B;
  int* wi = reinterpret_cast<int*>(wv + kNumConsumerWarps * B);
  unsigned& last = *reinterpret_cast<unsigned*>(wi + kNumConsumerWarps * B);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const Phase P0 = make_phase(static_cast<const T*>(p.w) + (size_t)t0 * kTileRows * D, nullptr,
                              t1 - t0, kTileRows * D * tb, true);
  pdl_launch_dependents();
  if (warp == kNumConsumerWarps) {
    const Phase ph[1] = {P0};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  pdl_wait();
  rmsnorm_to_smem<T, XH>(xs, p.resid, static_cast<const T*>(p.norm_w), B, D, p.eps, red, tid);
  float bv[QB];
  int bi[QB];
#pragma unroll
  for (int b = 0; b < QB; ++b) {
    bv[b] = -INFINITY;
    bi[b] = 0x7fffffff;
  }
  int cnt = 0;
  tiled_gemv_phase<T, QB, XH>(P0, ring, warp, lane, tid, cnt, xs, D, B, rows, part,
                          [&](int row, int b, float s) {
                            const int v = kTileRows * t0 + row;
                            if (v >= V) return;
                            if (p.logits) p.logits[(size_t)b * V + v] = s;
#pragma unroll
                            for (int bb = 0; bb < QB; ++bb)
                              if (bb == b && better(s, v, bv[bb], bi[bb])) {
                                bv[bb] = s;
                                bi[bb] = v;
                              }
                          });
  // per-thread best -> warp best -> CTA candidate
#pragma unroll
  for (int b = 0; b < QB; ++b) {
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv[b], o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi[b], o);
      if (better(ov, oi, bv[b], bi[b])) {
        bv[b] = ov;
        bi[b] = oi;
      }
    }
    if (lane == 0 && b < B) {
      wv[warp * B + b] = bv[b];
      wi[warp * B + b] = bi[b];
    }
  }
  consumer_sync();
  if (tid < B) {
    float v = -INFINITY;
    int ix = 0x7fffffff;
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2)
      if (better(wv[w2 * B + tid], wi[w2 * B + tid], v, ix)) {
        v = wv[w2 * B + tid];
        ix = wi[w2 * B + tid];
      }
    p.cand_val[(size_t)i * B + tid] = v;
    p.cand_idx[(size_t)i * B + tid] = ix;
  }
  __threadfence();
  consumer_sync();
  if (tid == 0) last = (atomicAdd(p.ticket, 1u) == (unsigned)G - 1);
  consumer_sync();
  if (last) {
    __threadfence();
    // warp w reduces rows b = w, w + 8, ...: lanes load the candidates in
    // parallel (one round trip instead of G serial ones), then shuffles;
    // `better` is a total order, so the tree shape cannot change the winner
    for (int b = warp; b < B; b += kNumConsumerWarps) {
      float v = -INFINITY;
      int ix = 0x7fffffff;
      for (int c = lane; c < G; c += 32) {
        const float cv = __ldcg(&p.cand_val[(size_t)c * B + b]);
        const int ci = __ldcg(&p.cand_idx[(size_t)c * B + b]);
        if (better(cv, ci, v, ix)) {
          v = cv;
          ix = ci;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
        if (better(ov, oi, v, ix)) {
          v = ov;
          ix = oi;
        }
      }
      if (lane == 0) p.token_out[b] = ix;
    }
    if (tid == 0) {
      *p.ticket = 0;
      if (p.step_pos) *p.step_pos += 1;
    }
  }
}

template <typename T>
__global__ void embed_kernel(const T* table, const int* tokens, float* out, int B, int D) {
  pdl_launch_dependents();
  pdl_wait();
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < B * D; idx += gridDim.x * blockDim.x) {
    const int b = idx / D, d = idx % D;
    out[idx] = Elem<T>::to_f(table[(size_t)tokens[b] * D + d]);
  }
}

template <typename T, int QB>
static int launch_lm_inst(const LmParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = lm_head_kernel<T, QB>;
  if (const int rc = configure_kernel((const void*)kern, kMaxSmem, false)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  LaunchAttrs at(0, p.flags & CFB_PDL);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

int lm_head_argmax(const cfb_lm_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  const int tb = a->dtype;
  if (tb != CFB_F16 && tb != CFB_F32) return set_error(CFB_ERR_ARGUMENT, "bad dtype");
  if (a->batch < 1 || a->batch > 8) return set_error(CFB_ERR_DIMENSION, "lm batch must be in [1, 8]");
  if (a->hidden % 8) return set_error(CFB_ERR_DIMENSION, "hidden must be a multiple of 8");
  if (!a->resid || !a->norm_w || !a->w || !a->cand_val || !a->cand_idx || !a->ticket || !a->token_out)
    return set_error(CFB_ERR_ARGUMENT, "null pointer");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = a->grid > 0 ? a->grid : sms;
  if (grid > a->vocab / kTileRows) grid = a->vocab / kTileRows;
  if (grid < 1) grid = 1;
  int spw = tuned_spw();
  const int TV = (a->vocab + kTileRows - 1) / kTileRows;
  const int rows_max = kTileRows * ((TV + grid - 1) / grid);
  auto need = [&](int s) {
    return (size_t)ring_bytes(s) + 2 * kNumSlots * 8 + (size_t)a->batch * a->hidden * 4 +
           (size_t)kNumConsumerWarps * a->batch * rows_max * 4 + 3 * kNumConsumerWarps * a->batch * 4 + 16;
  };
  while (need(spw) > (size_t)kMaxSmem && spw > 1) --spw;
  const size_t smem = need(spw);
  if (smem > (size_t)kMaxSmem) return set_error(CFB_ERR_SMEM, "lm head needs too much smem");
  LmParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.V = a->vocab;
  p.flags = a->flags;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.eps = a->eps;
  p.resid = a->resid;
  p.norm_w = a->norm_w;
  p.w = a->w;
  p.logits = a->logits;
  p.cand_val = a->cand_val;
  p.cand_idx = a->cand_idx;
  p.ticket = a->ticket;
  p.token_out = a->token_out;
  p.step_pos = a->step_pos;
  if (tb == 2) {
    if (p.B == 1) return launch_lm_inst<__half, 1>(p, grid, smem, st);
    return launch_lm_inst<__half, 8>(p, grid, smem, st);
  }
  if (p.B == 1) return launch_lm_inst<float, 1>(p, grid, smem, st);
  return launch_lm_inst<float, 8>(p, grid, smem, st);
}

int embed(int dtype, const void* table, const int* tokens, float* out, int B, int D,
          cudaStream_t st, bool pdl) {
  if (!table || !tokens || !out) return set_error(CFB_ERR_ARGUMENT, "null pointer");
  const int threads = 256, blocks = (B * D + threads - 1) / threads;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  if (dtype == CFB_F16)
    CFB_CUDA(cudaLaunchKernelEx(&cfg, embed_kernel<__half>, static_cast<const __half*>(table), tokens,
                                out, B, D));
  else
    CFB_CUDA(cudaLaunchKernelEx(&cfg, embed_kernel<float>, static_cast<const float*>(table), tokens,
                                out, B, D));
  return CFB_OK;
}

}  // namespace cfb
