// Fused SwiGLU FFN decode kernel (one launch): [RMSNorm ->] gate/up GEMV ->
// SiLU(gate) * up -> down GEMV [-> + residual].
//
// Reference semantics: ffn_reference(z, w1, w2, w3, "silu")
// (pkg/src/clusterdec/oracle.py:112-131) = (silu(z w1^T) * (z w2^T)) w3^T.
// The reference has no fused counterpart; this kernel is the
// north-star "gate/up GEMV, SiLU*mul and down GEMV in one launch".
//
// Persistent grid of one CTA per SM.  Weights are row-tiled (gemv.cuh):
//   w_gu tile t = rows (w1[2t], w1[2t+1], w2[2t], w2[2t+1])   F/2 tiles of D
//   w_dn tile u = rows 4u..4u+3 of w3                          D/4 tiles of F
// CTA i owns gate/up tiles [i*T1/G, (i+1)*T1/G) and down tiles
// [i*T2/G, (i+1)*T2/G).  The activation vector crosses CTAs once, through
// global memory and a grid barrier; the producer warp keeps streaming this
// CTA's w3 tiles into the ring while the barrier is pending, so HBM never
// idles at the phase boundary.
//
// Decoder-block form: the residual entering the block is r = resid + the
// attention module's fixed-point head sum (accum), folded into the RMSNorm
// prologue; after the grid barrier every CTA re-zeroes accum for the output
// rows it owns, and writes out = r + FFN for those rows (out may alias
// resid).  Without CFB_RESID (tensor-parallel ranks > 0) it writes the
// partial FFN only, so a sum over ranks adds r exactly once.  With PDL the
// producer streams w_gu before griddepcontrol.wait.
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct FfnParams {
  int B, D, F, flags, spw, sleep_max;
  float eps;
  const void* x;          // [B][D] T (no CFB_NORM)
  const float* resid;     // [B][D] fp32
  unsigned long long* accum;  // [B][D] fixed-point attention head sum (nullable)
  const void* norm_w;     // [D] T
  const void* w_gu;       // row-tiled, F/2 tiles of D
  const void* w_dn;       // row-tiled, D/4 tiles of F
  void* act;              // [B][F] T workspace
  float* out;             // [B][D] fp32
  unsigned long long* barrier;  // [0] grid barrier, [1] dynamic tile counter (both monotonic)
  unsigned long long* trace;
  int pool;                     // gate/up tiles handed out dynamically (0: fully static)
};

// x (phase 0 input, B x D) and act (phase 1 input, B x F) are never live at
// the same time and share one fp32 region.
struct FfnLayout {
  int bars, x, gu, part, red, tag, total;
};

__host__ __device__ inline FfnLayout ffn_layout(int B, int D, int F, int G, int spw, bool xh) {
  FfnLayout L;
  const int t1 = (F / 2 + G - 1) / G, t2 = (D / 4 + G - 1) / G;  // max tiles per CTA
  const int rows = 4 * (t1 > t2 ? t1 : t2);
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.x = o;     o += ((B * (D > F ? D : F) * (xh ? 2 : 4) + 15) & ~15);
  L.gu = o;    o += ((B * 4 * t1 * 4 + 15) & ~15);
  L.part = o;  o += ((kNumConsumerWarps * B * rows * 4 + 15) & ~15);
  L.red = o;   o += (kNumConsumerWarps * B * 4 + 15) & ~15;
  L.tag = o;   o += kNumSlots * 4;  // dynamic pool: tile index per ring slot (-1: end)
  L.total = o;
  return L;
}

template <typename T, int QB, bool XH>
__global__ void __launch_bounds__(kThreads, 1) ffn_swiglu_kernel(const FfnParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  const int B = p.B, D = p.D, F = p.F, G = gridDim.x, i = blockIdx.x;
  const FfnLayout L = ffn_layout(B, D, F, G, p.spw, XH);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // gate/up tiles: a static prefix [0, T1s) split evenly, then a pool of
  // p.pool tiles grabbed one at a time by the producer lanes (work stealing
  // absorbs the few-us spread of per-SM HBM throughput before the barrier)
  const int T1 = F / 2, T2 = D / 4, T1s = T1 - p.pool;
  const int a0 = (int)((long long)i * T1s / G), a1 = (int)((long long)(i + 1) * T1s / G);
  const int u0 = (int)((long long)i * T2 / G), u1 = (int)((long long)(i + 1) * T2 / G);
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const Phase P0 = make_phase(static_cast<const T*>(p.w_gu) + (size_t)a0 * 4 * D, nullptr, a1 - a0,
                              4 * D * tb, true);
  const Phase P1 = make_phase(static_cast<const T*>(p.w_dn) + (size_t)u0 * 4 * F, nullptr, u1 - u0,
                              4 * F * tb, true);
  const int tileB = 4 * D * tb, npc = (tileB + kSlotBytes - 1) / kSlotBytes;  // pieces per tile
  int* tag = reinterpret_cast<int*>(smem + L.tag);
  pdl_launch_dependents();
  if (warp == kNumConsumerWarps) {
    const uint64_t pol = policy_evict_first();
    int c = 0;
    {
      const Phase ph[1] = {P0};
      produce_all(ph, ring, lane, pol, c);
    }
    if (p.pool > 0) {
      // launch epoch: completed grid barriers / G; each lane makes exactly one
      // failing grab, so a launch adds pool + 8 G.  After the PDL wait every
      // earlier FFN launch has completed (when the grid leaves SMs idle, this
      // launch's CTAs can otherwise start while the previous FFN still runs)
      pdl_wait();
      const unsigned long long per = (unsigned long long)p.pool + 8ull * G;
      const unsigned long long base = (ld_acquire_u64(p.barrier) / (unsigned long long)G) * per;
      bool done = lane >= kNumConsumerWarps;
      int cur = 0, piece = npc, nap = 32;
      while (true) {
        bool issued = false;
        if (!done) {
          const int sl = lane * ring.spw + (c % ring.spw);
          if (mbar_test(&ring.empty[sl], ((c / ring.spw) & 1) ^ 1)) {
            if (piece == npc) {
              const long long t = (long long)(atomicAdd(p.barrier + 1, 1ull) - base);
              if (t >= p.pool) {  // pool exhausted: sentinel slot
                tag[sl] = -1;
                mbar_arrive(&ring.full[sl]);
                done = true;
              } else {
                cur = T1s + (int)t;
                piece = 0;
              }
            }
            if (!done) {
              const int b0 = piece * kSlotBytes, nb = min(kSlotBytes, tileB - b0);
              tag[sl] = cur;
              mbar_arrive_expect_tx(&ring.full[sl], (uint32_t)nb);
              bulk_g2s(ring.slot(sl), static_cast<const char*>(p.w_gu) + (size_t)cur * tileB + b0, nb,
                       &ring.full[sl], pol);
              ++piece;
            }
            ++c;
            issued = true;
          }
        }
        if (__all_sync(0xffffffffu, done)) break;
        if (__any_sync(0xffffffffu, issued)) {
          nap = 32;
        } else {
          __nanosleep(nap);
          nap = min(2 * nap, ring.sleep_max);
        }
      }
    }
    const Phase ph[1] = {P1};
    produce_all(ph, ring, lane, pol, c);
    return;
  }
  pdl_wait();
  unsigned long long* tr = p.trace ? p.trace + (size_t)i * 8 : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer();
  XElem<XH>* xs = reinterpret_cast<XElem<XH>*>(smem + L.x);
  float* gu = reinterpret_cast<float*>(smem + L.gu);  // [B][4*(a1-a0)]
  float* part = reinterpret_cast<float*>(smem + L.part);
  float* red = reinterpret_cast<float*>(smem + L.red);
  const int rows0 = 4 * (a1 - a0);

  if ((p.flags & CFB_NORM) && p.accum) {
    const float* resid = p.resid;
    const unsigned long long* acc = p.accum;
    rmsnorm_to_smem_ld<T, XH>(
        xs,
        [&](int b, int v) {
          const float4 r = reinterpret_cast<const float4*>(resid + (size_t)b * D)[v];
          const ulonglong2 a0 = __ldcg(reinterpret_cast<const ulonglong2*>(acc + (size_t)b * D) + 2 * v);
          const ulonglong2 a1 = __ldcg(reinterpret_cast<const ulonglong2*>(acc + (size_t)b * D) + 2 * v + 1);
          return make_float4(__fadd_rn(r.x, fixed_to_float(a0.x)), __fadd_rn(r.y, fixed_to_float(a0.y)),
                             __fadd_rn(r.z, fixed_to_float(a1.x)), __fadd_rn(r.w, fixed_to_float(a1.y)));
        },
        static_cast<const T*>(p.norm_w), B, D, p.eps, red, tid);
  } else if (p.flags & CFB_NORM) {
    rmsnorm_to_smem<T, XH>(xs, p.resid, static_cast<const T*>(p.norm_w), B, D, p.eps, red, tid);
  } else
    load_act_to_smem<T, XH>(xs, static_cast<const T*>(p.x), B, D, tid);

  if (tr && tid == 0) tr[1] = globaltimer();
  int cnt = 0;
  tiled_gemv_phase<T, QB, XH>(P0, ring, warp, lane, tid, cnt, xs, D, B, rows0, part,
                          [&](int row, int b, float v) { gu[b * rows0 + row] = v; });
  consumer_sync();
  T* act_g = static_cast<T*>(p.act);
  const int nf = 2 * (a1 - a0);
  for (int idx = tid; idx < B * nf; idx += kConsumerThreads) {
    const int b = idx / nf, j = idx % nf;           // f = 2*a0 + j
    const int t = j >> 1, e = j & 1;                // tile rows: g0 g1 u0 u1
    const float g = gu[b * rows0 + 4 * t + e], u = gu[b * rows0 + 4 * t + 2 + e];
    const float sl = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
    act_g[(size_t)b * F + 2 * a0 + j] = Elem<T>::from_f(__fmul_rn(sl, u));
  }
  if (p.pool > 0) {
    // dynamic pool: whole tiles (npc pieces in this warp's consecutive slots);
    // lanes 0..3 accumulate rows (gate 2t, gate 2t+1, up 2t, up 2t+1)
    while (true) {
      const int sl = warp * ring.spw + (cnt % ring.spw);
      mbar_wait(&ring.full[sl], (cnt / ring.spw) & 1);
      const int t = tag[sl];
      if (t < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[sl]);
        ++cnt;
        break;
      }
      float rowsum = 0.f;
      for (int pc = 0; pc < npc; ++pc) {
        const int s2 = warp * ring.spw + (cnt % ring.spw);
        if (pc > 0) mbar_wait(&ring.full[s2], (cnt / ring.spw) & 1);
        Item it;
        it.unit0 = 0;
        it.nunits = 1;
        it.piece = pc;
        it.byte0 = pc * kSlotBytes;
        it.bytes = min(kSlotBytes, tileB - it.byte0);
        tile_item<T, QB, XH>(P0, it, ring.slot(s2), xs, D, B, lane,
                             [&](int row, const float (&sm)[QB]) { rowsum += sm[0]; });
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[s2]);
        ++cnt;
      }
      // lane e (0, 1): gate from lane e, up from lane 2 + e
      const float up = __shfl_sync(0xffffffffu, rowsum, (lane & 1) + 2);
      if (lane < 2) {
        const float sl2 = __fdiv_rn(rowsum, __fadd_rn(1.0f, expf(-rowsum)));
        act_g[2 * t + lane] = Elem<T>::from_f(__fmul_rn(sl2, up));
      }
    }
  }
  if (tr && tid == 0) tr[2] = globaltimer();
  grid_barrier(p.barrier, tid);
  if (tr && tid == 0) tr[3] = globaltimer();
  load_act_to_smem<T, XH>(xs, act_g, B, F, tid);
  if (tr && tid == 0) tr[4] = globaltimer();

  const int rows1 = 4 * (u1 - u0);
  tiled_gemv_phase<T, QB, XH>(P1, ring, warp, lane, tid, cnt, xs, F, B, rows1, part,
                          [&](int row, int b, float v) {
                            const size_t c = (size_t)b * D + 4 * u0 + row;
                            if (p.flags & CFB_RESID) {
                              float r = p.resid[c];
                              if (p.accum) {
                                r = __fadd_rn(r, fixed_to_float(__ldcg(p.accum + c)));
                                p.accum[c] = 0ull;  // every CTA read it before the barrier
                              }
                              v = __fadd_rn(r, v);
                            } else if (p.accum) {
                              p.accum[c] = 0ull;  // tensor-parallel rank > 0: partial only
                            }
                            p.out[c] = v;
                          });
  if (tr && tid == 0) tr[5] = globaltimer();
}

template <typename T, int QB, bool XH>
static int launch_ffn_inst(const FfnParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = ffn_swiglu_kernel<T, QB, XH>;
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

int ffn_decode(const cfb_ffn_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  const int tb = a->dtype;
  if (tb != CFB_F16 && tb != CFB_F32) return set_error(CFB_ERR_ARGUMENT, "bad dtype");
  if (a->batch < 1 || a->batch > 8) return set_error(CFB_ERR_DIMENSION, "ffn batch must be in [1, 8]");
  if (a->hidden % 8 || a->inter % 8)
    return set_error(CFB_ERR_DIMENSION, "hidden and inter must be multiples of 8");
  if (!a->w_gu || !a->w_dn || !a->act || !a->out || !a->barrier)
    return set_error(CFB_ERR_ARGUMENT, "null weight / workspace pointer");
  if ((a->flags & CFB_NORM) ? (!a->resid || !a->norm_w) : !a->x)
    return set_error(CFB_ERR_ARGUMENT, "missing activation input");
  if ((a->flags & CFB_RESID) && !a->resid) return set_error(CFB_ERR_ARGUMENT, "CFB_RESID needs resid");
  if (a->accum && !(a->flags & CFB_NORM))
    return set_error(CFB_ERR_ARGUMENT, "accum needs CFB_NORM");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = a->grid > 0 ? a->grid : sms;
  grid = grid > sms ? sms : grid;  // grid barrier: every CTA must be co-resident
  if (grid > a->hidden / 4) grid = a->hidden / 4;
  if (grid > a->inter / 2) grid = a->inter / 2;
  // fp16 activations in smem for fp16 weights (FHFMA GEMV path)
  const bool xh = tb == 2;
  int spw = tuned_spw();
  FfnLayout L = ffn_layout(a->batch, a->hidden, a->inter, grid, spw, xh);
  while (L.total > kMaxSmem && spw > 1) L = ffn_layout(a->batch, a->hidden, a->inter, grid, --spw, xh);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "ffn schedule needs %d B of shared memory (max %d)", L.total,
                     kMaxSmem);
  FfnParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.F = a->inter;
  p.flags = a->flags;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.eps = a->eps;
  p.x = a->x;
  p.resid = a->resid;
  p.accum = a->accum;
  p.norm_w = a->norm_w;
  p.w_gu = a->w_gu;
  p.w_dn = a->w_dn;
  p.act = a->act;
  p.out = a->out;
  p.barrier = a->barrier;
  p.trace = a->trace;
  // dynamic gate/up pool (batch 1, engine launches): ~4 tiles per CTA
  p.pool = (a->batch == 1 && (a->flags & CFB_DYN_POOL)) ? min(4 * grid, a->inter / 2 / 4) : 0;
  const size_t smem = L.total;
  if (tb == 2) {
    if (p.B == 1) return launch_ffn_inst<__half, 1, true>(p, grid, smem, st);
    if (p.B == 2) return launch_ffn_inst<__half, 2, true>(p, grid, smem, st);
    if (p.B <= 4) return launch_ffn_inst<__half, 4, true>(p, grid, smem, st);
    return launch_ffn_inst<__half, 8, true>(p, grid, smem, st);
  }
  if (p.B == 1) return launch_ffn_inst<float, 1, false>(p, grid, smem, st);
  if (p.B <= 4) return launch_ffn_inst<float, 4, false>(p, grid, smem, st);
  return launch_ffn_inst<float, 8, false>(p, grid, smem, st);
}

}  // namespace cfb
