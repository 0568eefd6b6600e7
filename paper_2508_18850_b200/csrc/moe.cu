// Fused DeepSeek-V2 MoE decode kernel (one launch): [residual + attention
// head sum -> RMSNorm ->] router GEMV -> softmax top-k -> shared + routed
// expert SwiGLU GEMVs -> weighted sum [-> + residual].
//
// Semantics: DeepseekV2Moe.forward of transformers (greedy softmax top-k,
// norm_topk_prob False, routed_scaling_factor, shared experts as one MLP of
// width n_shared * F_e), restated in oracle/deepseek_port.py:moe with the
// SwiGLU activation stored as fp16.  The reference package has no MoE
// (SPEC.md:12, :366); this is the north-star "fused MoE top-k router plus
// expert GEMV" of config #3.
//
// Work split (persistent grid, one CTA per SM, no grid barrier before the
// last step).  The intermediate dimension of every expert is cut into
// groups of 8 f; a CTA owns a contiguous range of shared-expert groups and
// a contiguous range of routed groups (in the concatenation of the selected
// experts, ascending expert id), balanced so that both together differ by
// at most one group across CTAs.  For each of its groups a CTA computes the
// 8 gate/up pairs (row-tiled GEMV over D), the SwiGLU activations, and the
// down-projection contribution of those 8 columns to all D outputs
// (split-K), which it adds into a 64-bit fixed-point accumulator with
// red.global.add - integer adds, so the result is independent of CTA order.
// A final grid barrier lets every CTA finish its slice of the output
// (out = resid + attention sum + MoE sum) and re-zero the accumulators.
//
// Router: every CTA computes all E logits itself from the (L2-resident)
// router matrix while its producer warp already streams the shared experts,
// so no CTA waits on another for routing; the selected experts reach the
// producer through a shared-memory mbarrier.
//
// Weight layouts (fp16, prepared by moe.py):
//   w_router [E][D]
//   w_gu     [E][F_e/2 tiles][D/8 chunks][4 rows][8]  tile t = (gate 2t, gate 2t+1,
//                                                     up 2t, up 2t+1)  (FFN layout)
//   w_dn     [E][F_e/8 groups][Q][8 f][D/Q]           W_down^T blocks, Q = max(1, D/512)
//   s_gu / s_dn: the shared experts in the same layouts (F_s = n_shared * F_e).
// A down block is 8 f x D/Q columns (8 KB at D/Q = 512); consumer warp w
// always gets segment w % Q, so its lanes own fixed output columns and
// accumulate in registers across all its blocks.
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

constexpr int kMoeMaxExperts = 256;
constexpr int kMoeMaxTopK = 16;
constexpr int kMoeMaxBatch = 4;

struct MoeParams {
  int B, D, E, K, Fe, Fs, Q, flags, spw, sleep_max;
  float eps, scale;
  const __half* x;
  const float* resid;
  unsigned long long* accum_in;  // attention fixed-point head sum (nullable)
  const __half* norm_w;
  const __half* w_router;
  const __half* w_gu;
  const __half* w_dn;
  const __half* s_gu;
  const __half* s_dn;
  unsigned long long* accum;  // [B][D] MoE fixed-point sum (zero; re-zeroed)
  float* out;
  int* route_idx;
  float* route_w;
  unsigned long long* barrier;
};

struct MoeLayout {
  int bars, xs, logit, sel, slot, gw, tk, gu, part, act, dpart, red, total;
  int max_groups, umax;
};

__host__ __device__ inline int moe_r16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline MoeLayout moe_layout(int B, int D, int E, int K, int Fe, int Fs, int Q,
                                                int G, int spw) {
  MoeLayout L;
  const int Gs = Fs / 8, Ge = Fe / 8;
  L.umax = B * K < E ? B * K : E;
  const int Tt = Gs + L.umax * Ge;
  L.max_groups = (Tt + G - 1) / G + 1;
  int o = ring_bytes(spw);
  L.bars = o;  o += moe_r16((2 * kNumSlots + 1) * 8);
  L.xs = o;    o += moe_r16(B * D * 2);
  L.logit = o; o += moe_r16(B * E * 4);
  L.sel = o;   o += moe_r16(E);
  L.slot = o;  o += moe_r16((L.umax + 1) * 4);
  L.gw = o;    o += moe_r16(B * L.umax * 4);
  L.tk = o;    o += moe_r16(2 * B * K * 4);
  L.gu = o;    o += moe_r16(B * 16 * L.max_groups * 4);
  L.part = o;  o += moe_r16(kNumConsumerWarps * B * 16 * L.max_groups * 4);
  L.act = o;   o += moe_r16(2 * B * 8 * L.max_groups * 4);
  L.dpart = o; o += moe_r16((8 / Q) * B * D * 4);
  L.red = o;   o += moe_r16(kNumConsumerWarps * B * 4);
  L.total = o;
  return L;
}

// Group ranges of CTA i: shared [s0, s1), routed [r0, r1) of the
// concatenation of U selected experts (Ge groups each).  t = s + r is split
// evenly, so every CTA gets floor or ceil of (Gs + U*Ge) / G groups.
struct MoeRange {
  int s0, s1, r0, r1;
};
__device__ __forceinline__ MoeRange moe_range(int i, int G, int Gs, int Tr) {
  const long long Tt = (long long)Gs + Tr;
  MoeRange m;
  m.s0 = (int)((long long)i * Gs / G);
  m.s1 = (int)((long long)(i + 1) * Gs / G);
  m.r0 = (int)((long long)i * Tt / G) - m.s0;
  m.r1 = (int)((long long)(i + 1) * Tt / G) - m.s1;
  return m;
}

// top-k (descending logit, ties to the lower expert index) and the softmax
// probability of each selected expert, for one token row; warp-wide.
__device__ __forceinline__ void topk_row(const float* lg, int E, int K, float scale, int lane,
                                         int* idx_out, float* w_out) {
  constexpr int kPer = kMoeMaxExperts / 32;
  float v[kPer];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = lane + 32 * k;
    v[k] = e < E ? lg[e] : -INFINITY;
    m = fmaxf(m, v[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (lane + 32 * k < E) s += expf(v[k] - m);
  s = warp_allsum(s);
  unsigned taken = 0;
  for (int j = 0; j < K; ++j) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = lane + 32 * k;
      if (e < E && !(taken >> k & 1u) && (v[k] > bv || (v[k] == bv && e < bi))) {
        bv = v[k];
        bi = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    if (lane == 0) {
      idx_out[j] = bi;
      w_out[j] = __fmul_rn(__fdiv_rn(expf(bv - m), s), scale);
    }
  }
}

template <int QB>
__global__ void __launch_bounds__(kThreads, 1) moe_kernel(const MoeParams p) {
  extern __shared__ __align__(128) char smem[];
  const int B = p.B, D = p.D, E = p.E, K = p.K, Q = p.Q, G = gridDim.x, i = blockIdx.x;
  const MoeLayout L = moe_layout(B, D, E, K, p.Fe, p.Fs, Q, G, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* route_bar = bars + 2 * kNumSlots;
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Gs = p.Fs / 8, Ge = p.Fe / 8;
  const int Wd = D / Q;                        // columns per down segment
  const int tileB = 4 * D * 2;                 // gate/up tile: 4 rows x D fp16
  const int blkB = 16 * Wd;                    // down block: 8 rows x Wd fp16
  const size_t eGu = (size_t)(p.Fe / 2) * 4 * D, eDn = (size_t)Ge * 8 * D;  // elements per expert
  int* slot_e = reinterpret_cast<int*>(smem + L.slot);  // [umax] expert ids, [umax] = U
  if (tid == 0) {
    ring_init(ring);
    mbar_init(route_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const MoeRange rs = moe_range(i, G, Gs, 0);  // shared part is routing-independent
  const Phase GUs = make_phase(p.s_gu + (size_t)rs.s0 * 4 * 4 * D, nullptr, 4 * (rs.s1 - rs.s0),
                               tileB, true);
  const Phase DNs = make_phase(p.s_dn + (size_t)rs.s0 * 8 * D, nullptr, Q * (rs.s1 - rs.s0), blkB);
  auto routed_phase = [&](const MoeRange& m, int u, bool down) {
    const int ga = max(m.r0, u * Ge) - u * Ge, gb = min(m.r1, (u + 1) * Ge) - u * Ge;
    const int e = slot_e[u];
    if (down)
      return make_phase(p.w_dn + e * eDn + (size_t)ga * 8 * D, nullptr, Q * (gb - ga), blkB);
    return make_phase(p.w_gu + e * eGu + (size_t)ga * 4 * 4 * D, nullptr, 4 * (gb - ga), tileB, true);
  };
  pdl_launch_dependents();

  if (warp == kNumConsumerWarps) {  // producer
    const uint64_t pol = policy_evict_first();
    int c = 0;
    const Phase ps[2] = {GUs, DNs};
    produce_all(ps, ring, lane, pol, c);
    mbar_wait(route_bar, 0);
    const int U = slot_e[L.umax];
    const MoeRange m = moe_range(i, G, Gs, U * Ge);
    for (int pass = 0; pass < 2; ++pass)
      for (int u = m.r0 / Ge; u < U && u * Ge < m.r1; ++u) {
        const Phase ph[1] = {routed_phase(m, u, pass == 1)};
        produce_all(ph, ring, lane, pol, c);
      }
    return;
  }

  pdl_wait();
  __half* xs = reinterpret_cast<__half*>(smem + L.xs);
  float* logit = reinterpret_cast<float*>(smem + L.logit);
  unsigned char* sel = reinterpret_cast<unsigned char*>(smem + L.sel);
  float* gw = reinterpret_cast<float*>(smem + L.gw);     // [B][umax]
  float* gu = reinterpret_cast<float*>(smem + L.gu);     // [B][16 * groups]
  float* part = reinterpret_cast<float*>(smem + L.part);
  float* act = reinterpret_cast<float*>(smem + L.act);   // [B][8 * groups] (x2: shared, routed)
  float* dpart = reinterpret_cast<float*>(smem + L.dpart);
  float* red = reinterpret_cast<float*>(smem + L.red);

  // 0. activations: x = f16(rmsnorm(resid [+ attention sum]) * g), or x
  if ((p.flags & CFB_NORM) && p.accum_in) {
    const float* resid = p.resid;
    const unsigned long long* acc = p.accum_in;
    rmsnorm_to_smem_ld<__half, true>(
        xs,
        [&](int b, int v) {
          const float4 r = reinterpret_cast<const float4*>(resid + (size_t)b * D)[v];
          const ulonglong2 a0 = __ldcg(reinterpret_cast<const ulonglong2*>(acc + (size_t)b * D) + 2 * v);
          const ulonglong2 a1 = __ldcg(reinterpret_cast<const ulonglong2*>(acc + (size_t)b * D) + 2 * v + 1);
          return make_float4(__fadd_rn(r.x, fixed_to_float(a0.x)), __fadd_rn(r.y, fixed_to_float(a0.y)),
                             __fadd_rn(r.z, fixed_to_float(a1.x)), __fadd_rn(r.w, fixed_to_float(a1.y)));
        },
        p.norm_w, B, D, p.eps, red, tid);
  } else if (p.flags & CFB_NORM) {
    rmsnorm_to_smem<__half, true>(xs, p.resid, p.norm_w, B, D, p.eps, red, tid);
  } else {
    load_act_to_smem<__half, true>(xs, p.x, B, D, tid);
  }

  // 1. router logits (fp32), every CTA: warp w takes experts w, w+8, ...
  {
    const int nch = D / 8;
    for (int e0 = warp; e0 < E; e0 += 2 * kNumConsumerWarps) {
      const int e1 = e0 + kNumConsumerWarps;
      float a0[QB], a1[QB];
#pragma unroll
      for (int b = 0; b < QB; ++b) a0[b] = a1[b] = 0.f;
      const uint4* r0 = reinterpret_cast<const uint4*>(p.w_router + (size_t)e0 * D);
      const uint4* r1 = reinterpret_cast<const uint4*>(p.w_router + (size_t)(e1 < E ? e1 : e0) * D);
      for (int c0 = 0; c0 < nch; c0 += 32 * 4) {
        uint4 w0[4], w1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = c0 + lane + 32 * k;
          w0[k] = c < nch ? __ldg(r0 + c) : make_uint4(0, 0, 0, 0);
          w1[k] = c < nch ? __ldg(r1 + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = c0 + lane + 32 * k;
          if (c < nch) {
#pragma unroll
            for (int b = 0; b < QB; ++b) {
              if (b < B) {
                const uint4 xv = lds128(xs + (size_t)b * D + c * 8);
                const uint32_t xr[4] = {xv.x, xv.y, xv.z, xv.w};
                const uint32_t q0[4] = {w0[k].x, w0[k].y, w0[k].z, w0[k].w};
                const uint32_t q1[4] = {w1[k].x, w1[k].y, w1[k].z, w1[k].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  a0[b] = fma_f16_hi(q0[j], xr[j], fma_f16_lo(q0[j], xr[j], a0[b]));
                  a1[b] = fma_f16_hi(q1[j], xr[j], fma_f16_lo(q1[j], xr[j], a1[b]));
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < QB; ++b) {
        if (b < B) {
          const float s0 = warp_allsum(a0[b]), s1 = warp_allsum(a1[b]);
          if (lane == 0) {
            logit[b * E + e0] = s0;
            if (e1 < E) logit[b * E + e1] = s1;
          }
        }
      }
    }
  }
  for (int e = tid; e < E; e += kConsumerThreads) sel[e] = 0;
  consumer_sync();

  // 2. top-k per token, union of the selected experts (ascending id), gate weights
  if (warp == 0) {
    int* s_idx = reinterpret_cast<int*>(smem + L.tk);
    float* s_w = reinterpret_cast<float*>(s_idx + B * K);
    for (int b = 0; b < B; ++b) topk_row(logit + b * E, E, K, p.scale, lane, s_idx + b * K, s_w + b * K);
    __syncwarp();
    for (int t = lane; t < B * K; t += 32) sel[s_idx[t]] = 1;
    __syncwarp();
    int U = 0;
    for (int base = 0; base < E; base += 32) {
      const bool f = base + lane < E && sel[base + lane];
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) slot_e[U + __popc(bal & ((1u << lane) - 1u))] = base + lane;
      U += __popc(bal);
    }
    __syncwarp();
    for (int t = lane; t < B * U; t += 32) gw[(t / U) * L.umax + t % U] = 0.f;
    __syncwarp();
    for (int t = lane; t < B * K; t += 32) {
      const int b = t / K, e = s_idx[t];
      int u = 0;
      while (slot_e[u] != e) ++u;
      gw[b * L.umax + u] = s_w[t];
    }
    if (lane == 0) slot_e[L.umax] = U;
    if (i == 0 && p.route_idx)
      for (int t = lane; t < B * K; t += 32) {
        p.route_idx[t] = s_idx[t];
        if (p.route_w) p.route_w[t] = s_w[t];
      }
  }
  consumer_sync();
  if (tid == 0) mbar_arrive(route_bar);
  const int U = slot_e[L.umax];
  const MoeRange m = moe_range(i, G, Gs, U * Ge);

  // 3. gate/up GEMV over a phase, SwiGLU, scaled activations into act_dst
  int cnt = 0;
  auto gate_up = [&](const Phase& P, int n_groups, float* act_dst, int act_ld, int f_off,
                     const float* wgt /* [B] or null: weight 1 */) {
    const int rows = 16 * n_groups;
    tiled_gemv_phase<__half, QB, true>(P, ring, warp, lane, tid, cnt, xs, D, B, rows, part,
                                       [&](int row, int b, float v) { gu[b * rows + row] = v; });
    consumer_sync();
    for (int t = tid; t < B * 8 * n_groups; t += kConsumerThreads) {
      const int b = t / (8 * n_groups), j = t % (8 * n_groups);  // f = 2*tile + e
      const int tl = j >> 1, e = j & 1;
      const float g = gu[b * rows + 4 * tl + e], uu = gu[b * rows + 4 * tl + 2 + e];
      const float a = __half2float(__float2half_rn(__fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), uu)));
      act_dst[b * act_ld + f_off + j] = wgt ? __fmul_rn(wgt[b * L.umax], a) : a;
    }
    consumer_sync();
  };

  // 4. split-K down projection of a phase's blocks: warp w owns segment w % Q
  constexpr int kCpl = 2;  // 16-byte chunks per lane per block row (Wd <= 512)
  float acc[QB][kCpl][8];
  auto zero_acc = [&] {
#pragma unroll
    for (int b = 0; b < QB; ++b)
#pragma unroll
      for (int j = 0; j < kCpl; ++j)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[b][j][e] = 0.f;
  };
  auto down = [&](const Phase& P, const float* a_src, int act_ld, int g_off) {
    const int nch = Wd / 8;
    consume_phase(P, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
      for (int uu = 0; uu < it.nunits; ++uu) {
        const int unit = it.unit0 + uu;
        const int gl = unit / Q + g_off;  // local group (seg = unit % Q == warp % Q)
        const char* blk = slot + (size_t)uu * blkB;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          float av[QB];
#pragma unroll
          for (int b = 0; b < QB; ++b) av[b] = b < B ? a_src[b * act_ld + 8 * gl + r] : 0.f;
#pragma unroll
          for (int j = 0; j < kCpl; ++j) {
            const int c = lane + 32 * j;
            if (c < nch) {
              const uint4 wv = lds128(blk + ((size_t)r * nch + c) * 16);
              float wf[8];
              Elem<__half>::unpack(wv, wf);
#pragma unroll
              for (int b = 0; b < QB; ++b)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[b][j][e] = fmaf(wf[e], av[b], acc[b][j][e]);
            }
          }
        }
      }
    });
  };
  auto flush = [&](bool add) {  // registers -> dpart[warp / Q][b][segment columns]
    float* dst = dpart + (size_t)(warp / Q) * B * D + (warp % Q) * Wd;
    const int nch = Wd / 8;
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      if (b < B) {
#pragma unroll
        for (int j = 0; j < kCpl; ++j) {
          const int c = lane + 32 * j;
          if (c < nch) {
            float4* d4 = reinterpret_cast<float4*>(dst + (size_t)b * D + c * 8);
            float4 v0 = make_float4(acc[b][j][0], acc[b][j][1], acc[b][j][2], acc[b][j][3]);
            float4 v1 = make_float4(acc[b][j][4], acc[b][j][5], acc[b][j][6], acc[b][j][7]);
            if (add) {
              const float4 o0 = d4[0], o1 = d4[1];
              v0 = make_float4(o0.x + v0.x, o0.y + v0.y, o0.z + v0.z, o0.w + v0.w);
              v1 = make_float4(o1.x + v1.x, o1.y + v1.y, o1.z + v1.z, o1.w + v1.w);
            }
            d4[0] = v0;
            d4[1] = v1;
          }
        }
      }
    }
  };

  float* act_s = act;
  float* act_r = act + B * 8 * L.max_groups;
  const int ns = rs.s1 - rs.s0, nr = m.r1 - m.r0;
  // shared experts
  gate_up(GUs, ns, act_s, 8 * L.max_groups, 0, nullptr);
  zero_acc();
  down(DNs, act_s, 8 * L.max_groups, 0);
  flush(false);
  // routed experts (this CTA's slice of the selected experts' concatenation)
  for (int u = m.r0 / Ge; u < U && u * Ge < m.r1; ++u) {
    const int ga = max(m.r0, u * Ge);
    gate_up(routed_phase(m, u, false), min(m.r1, (u + 1) * Ge) - ga, act_r, 8 * L.max_groups,
            8 * (ga - m.r0), gw + u);
  }
  zero_acc();
  for (int u = m.r0 / Ge; u < U && u * Ge < m.r1; ++u)
    down(routed_phase(m, u, true), act_r, 8 * L.max_groups, max(m.r0, u * Ge) - m.r0);
  flush(true);
  consumer_sync();
  (void)nr;

  // 5. this CTA's split-K partial into the fixed-point accumulator
  const int nparts = 8 / Q;
  for (int t = tid; t < B * D; t += kConsumerThreads) {
    float v = 0.f;
    for (int s = 0; s < nparts; ++s) v += dpart[(size_t)s * B * D + t];
    red_add_fixed(p.accum + t, v);
  }
  grid_barrier(p.barrier, tid);

  // 6. finish: out = [resid + attention sum +] MoE sum for this CTA's slice
  const int n = B * D, o0 = (int)((long long)i * n / G), o1 = (int)((long long)(i + 1) * n / G);
  for (int t = o0 + tid; t < o1; t += kConsumerThreads) {
    float v = fixed_to_float(__ldcg(p.accum + t));
    p.accum[t] = 0ull;
    if (p.flags & CFB_RESID) {
      float r = p.resid[t];
      if (p.accum_in) {
        r = __fadd_rn(r, fixed_to_float(__ldcg(p.accum_in + t)));
        p.accum_in[t] = 0ull;
      }
      v = __fadd_rn(r, v);
    }
    p.out[t] = v;
  }
}

template <int QB>
static int launch_moe_inst(const MoeParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = moe_kernel<QB>;
  static bool configured = false;
  if (!configured) {
    CFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    configured = true;
  }
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

int moe_segments(int hidden) { return hidden >= 512 ? hidden / 512 : 1; }

int moe_decode(const cfb_moe_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->dtype != CFB_F16) return set_error(CFB_ERR_DIMENSION, "the MoE kernel is fp16 only");
  if (a->batch < 1 || a->batch > kMoeMaxBatch)
    return set_error(CFB_ERR_DIMENSION, "moe batch must be in [1, %d]", kMoeMaxBatch);
  const int D = a->hidden, E = a->n_experts, K = a->top_k, Fe = a->inter, Fs = a->shared_inter;
  if (E < 1 || E > kMoeMaxExperts) return set_error(CFB_ERR_DIMENSION, "n_experts must be in [1, 256]");
  if (K < 1 || K > kMoeMaxTopK || K > E) return set_error(CFB_ERR_DIMENSION, "top_k must be in [1, min(16, E)]");
  if (Fe < 8 || Fe % 8 || Fs < 0 || Fs % 8)
    return set_error(CFB_ERR_DIMENSION, "expert widths must be multiples of 8 (inter >= 8)");
  if (D < 8 || D % 8 || (D > 512 && D % 512) || (D > 512 && 8 % (D / 512)))
    return set_error(CFB_ERR_DIMENSION, "hidden must be a multiple of 8 up to 512, or 512/1024/2048/4096");
  if (!a->w_router || !a->w_gu || !a->w_dn || (Fs && (!a->s_gu || !a->s_dn)) || !a->accum ||
      !a->out || !a->barrier)
    return set_error(CFB_ERR_ARGUMENT, "null weight / workspace pointer");
  if ((a->flags & CFB_NORM) ? (!a->resid || !a->norm_w) : !a->x)
    return set_error(CFB_ERR_ARGUMENT, "missing activation input");
  if ((a->flags & CFB_RESID) && !a->resid) return set_error(CFB_ERR_ARGUMENT, "CFB_RESID needs resid");
  if (a->accum_in && (a->flags & (CFB_NORM | CFB_RESID)) != (CFB_NORM | CFB_RESID))
    return set_error(CFB_ERR_ARGUMENT, "accum_in needs CFB_NORM | CFB_RESID");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int Ge = Fe / 8;
  int grid = a->grid > 0 ? a->grid : sms;
  if (grid > sms) grid = sms;         // grid barrier: every CTA co-resident
  if (grid > K * Ge) grid = K * Ge;   // routed groups >= grid keeps every range non-empty-ordered
  const int Q = moe_segments(D);
  int spw = tuned_spw();
  MoeLayout L = moe_layout(a->batch, D, E, K, Fe, Fs, Q, grid, spw);
  while (L.total > kMaxSmem && spw > 1) L = moe_layout(a->batch, D, E, K, Fe, Fs, Q, grid, --spw);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "moe schedule needs %d B of shared memory (max %d)", L.total, kMaxSmem);
  MoeParams p;
  p.B = a->batch;
  p.D = D;
  p.E = E;
  p.K = K;
  p.Fe = Fe;
  p.Fs = Fs;
  p.Q = Q;
  p.flags = a->flags;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.eps = a->eps;
  p.scale = a->routed_scale;
  p.x = static_cast<const __half*>(a->x);
  p.resid = a->resid;
  p.accum_in = a->accum_in;
  p.norm_w = static_cast<const __half*>(a->norm_w);
  p.w_router = static_cast<const __half*>(a->w_router);
  p.w_gu = static_cast<const __half*>(a->w_gu);
  p.w_dn = static_cast<const __half*>(a->w_dn);
  p.s_gu = static_cast<const __half*>(a->s_gu);
  p.s_dn = static_cast<const __half*>(a->s_dn);
  p.accum = a->accum;
  p.out = a->out;
  p.route_idx = a->route_idx;
  p.route_w = a->route_w;
  p.barrier = a->barrier;
  const size_t smem = L.total;
  if (p.B == 1) return launch_moe_inst<1>(p, grid, smem, st);
  if (p.B == 2) return launch_moe_inst<2>(p, grid, smem, st);
  return launch_moe_inst<4>(p, grid, smem, st);
}

}  // namespace cfb
