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
// The last CTA to finish (a ticket on a monotonic counter) writes the output
// (out = resid + attention sum + MoE sum) and re-zeroes the accumulators.
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
constexpr int kMoeChunk = 16;  // gate/up groups per GEMV phase (bounds the partial buffer)

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
  float* part;                // [grid][B*D] per-CTA partial sums (workspace)
  float* out;
  int* route_idx;
  float* route_w;
  unsigned long long* barrier;  // [0] finished CTAs, [1] published router rows (monotonic)
  float* logits;               // [B][E] router logits (workspace)
  unsigned long long* trace;  // [grid][16] %globaltimer phase stamps (profiling) or null
};

struct MoeLayout {
  int bars, rrow, xs, logit, slot, gw, tk, gu, part, act, dpart, red, total;
  int max_groups, umax, rrows;  // rrows: router rows prefetched into smem (0: read via L2)
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
  L.bars = o;  o += moe_r16((2 * kNumSlots + 3) * 8);
  const int rows = (E + G - 1) / G;
  L.rrows = rows * D * 2 <= 16384 ? rows : 0;
  L.rrow = o;  o += moe_r16(L.rrows * D * 2);
  L.xs = o;    o += moe_r16(B * D * 2);
  L.logit = o; o += moe_r16(2 * B * E * 4);
  L.slot = o;  o += moe_r16((L.umax + 1) * 4);
  L.gw = o;    o += moe_r16(B * L.umax * 4);
  L.tk = o;    o += moe_r16(2 * B * K * 4);
  L.gu = o;    o += moe_r16(B * 16 * kMoeChunk * 4);
  L.part = o;  o += moe_r16(kNumConsumerWarps * B * 16 * kMoeChunk * 4);
  L.act = o;   o += moe_r16(2 * B * 8 * L.max_groups * 2);
  L.dpart = o; o += moe_r16((8 / Q) * B * D * 4);
  L.red = o;   o += moe_r16(kNumConsumerWarps * (B > 2 ? B : 2) * 4);
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
  // 32-bit: (G <= 148) x (groups <= 32 * 256 * 16 / 8) stays far below 2^31, and a
  // 64-bit division is a slow software routine on the GPU
  const unsigned Tt = (unsigned)(Gs + Tr), g = (unsigned)G, u = (unsigned)i;
  MoeRange m;
  m.s0 = (int)(u * (unsigned)Gs / g);
  m.s1 = (int)((u + 1) * (unsigned)Gs / g);
  m.r0 = (int)(u * Tt / g) - m.s0;
  m.r1 = (int)((u + 1) * Tt / g) - m.s1;
  return m;
}

template <int QB>
__global__ void __launch_bounds__(kThreads, 1) moe_kernel(const MoeParams p) {
  extern __shared__ __align__(128) char smem[];
  const int B = p.B, D = p.D, E = p.E, K = p.K, Q = p.Q, G = gridDim.x, i = blockIdx.x;
  const MoeLayout L = moe_layout(B, D, E, K, p.Fe, p.Fs, Q, G, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* route_bar = bars + 2 * kNumSlots;
  uint64_t* rrow_bar = route_bar + 1;  // router rows landed in smem
  uint64_t* go_bar = rrow_bar + 1;     // consumers past griddepcontrol.wait: experts may stream
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Gs = p.Fs / 8, Ge = p.Fe / 8;
  const int Wd = D / Q;                        // columns per down segment
  const int tileB = 4 * D * 2;                 // gate/up tile: 4 rows x D fp16
  const int blkB = 16 * Wd;                    // down block: 8 rows x Wd fp16
  const size_t eGu = (size_t)Ge * 16 * D, eDn = (size_t)Ge * 8 * D;  // elements per expert
  int* slot_e = reinterpret_cast<int*>(smem + L.slot);  // [umax] expert ids, [umax] = U
  if (tid == 0) {
    ring_init(ring);
    mbar_init(route_bar, 1);
    mbar_init(rrow_bar, 1);
    mbar_init(go_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const MoeRange rs = moe_range(i, G, Gs, 0);  // shared part is routing-independent
  // phases: gate/up tiles of groups [g0, g0 + ng) (<= kMoeChunk groups per
  // phase, so the cross-warp partial buffer stays small), down blocks
  auto gu_phase = [&](const __half* base, int g0, int ng) {
    return make_phase(base + (size_t)g0 * 16 * D, nullptr, 4 * ng, tileB, true);
  };
  auto dn_phase = [&](const __half* base, int g0, int ng) {
    return make_phase(base + (size_t)g0 * 8 * D, nullptr, Q * ng, blkB);
  };
  // routed segment u of this CTA's range: expert slot_e[u], groups [ga, gb) of it
  auto seg = [&](const MoeRange& m, int u, int& ga, int& gb) {
    ga = max(m.r0, u * Ge) - u * Ge;
    gb = min(m.r1, (u + 1) * Ge) - u * Ge;
    return slot_e[u];
  };
  pdl_launch_dependents();

  if (warp == kNumConsumerWarps) {  // ------------------------------ producer
    const uint64_t pol = policy_evict_first();
    int c = 0;
    if (lane == 0 && L.rrows) {  // this CTA's router rows e = i, i + G, ... first
      int n = 0;
      for (int e = i; e < E; e += G) ++n;
      mbar_arrive_expect_tx(rrow_bar, (uint32_t)(n * D * 2));
      n = 0;
      for (int e = i; e < E; e += G, ++n)
        bulk_g2s(smem + L.rrow + (size_t)n * D * 2, p.w_router + (size_t)e * D, D * 2, rrow_bar,
                 policy_evict_last());  // router rows stay L2-resident across steps
    }
    // the expert stream starts once the consumers have issued their RMSNorm
    // loads: a 28 MB burst issued first would queue ahead of those loads
    if (lane == 0)
      while (!mbar_test(go_bar, 0)) __nanosleep(32);
    __syncwarp();
    for (int g = rs.s0; g < rs.s1; g += kMoeChunk) {
      const Phase ph[1] = {gu_phase(p.s_gu, g, min(kMoeChunk, rs.s1 - g))};
      produce_all(ph, ring, lane, pol, c);
    }
    {
      const Phase ph[1] = {dn_phase(p.s_dn, rs.s0, rs.s1 - rs.s0)};
      produce_all(ph, ring, lane, pol, c);
    }
    if (lane == 0)  // routing (consumer warps) -> expert list in smem
      while (!mbar_test(route_bar, 0)) __nanosleep(64);
    __syncwarp();
    const int U = slot_e[L.umax];
    const MoeRange m = moe_range(i, G, Gs, U * Ge);
    for (int u = m.r0 / Ge; u < U && u * Ge < m.r1; ++u) {
      int ga, gb;
      const int e = seg(m, u, ga, gb);
      for (int g = ga; g < gb; g += kMoeChunk) {
        const Phase ph[1] = {gu_phase(p.w_gu + e * eGu, g, min(kMoeChunk, gb - g))};
        produce_all(ph, ring, lane, pol, c);
      }
    }
    for (int u = m.r0 / Ge; u < U && u * Ge < m.r1; ++u) {
      int ga, gb;
      const int e = seg(m, u, ga, gb);
      const Phase ph[1] = {dn_phase(p.w_dn + e * eDn, ga, gb - ga)};
      produce_all(ph, ring, lane, pol, c);
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  pdl_wait();
  if (tid == 0) mbar_arrive(go_bar);
  unsigned long long* tr = p.trace ? p.trace + (size_t)i * 16 : nullptr;
  auto stamp = [&](int k) {  // %globaltimer ns (comparable across SMs and kernels)
    if (tr && tid == 0) tr[k] = globaltimer();
  };
  stamp(0);
  // launch epoch: barrier[0] counts finished CTAs (G per launch); no CTA of
  // this launch can finish before every CTA has published its router rows
  // (relaxed: the previous launch completed before pdl_wait returned; the
  // load's latency then overlaps the RMSNorm prologue instead of blocking it)
  const unsigned long long epoch =
      tid == 0 ? ld_relaxed_u64(p.barrier) / (unsigned long long)G : 0ull;
  __half* xs = reinterpret_cast<__half*>(smem + L.xs);
  float* lg = reinterpret_cast<float*>(smem + L.logit);   // [2][B][E]: logits, gate weights
  float* gw = reinterpret_cast<float*>(smem + L.gw);      // [B][umax]
  float* gu = reinterpret_cast<float*>(smem + L.gu);      // [B][16 * kMoeChunk]
  float* part = reinterpret_cast<float*>(smem + L.part);
  __half* act = reinterpret_cast<__half*>(smem + L.act);  // [2][B][8 * max_groups] fp16
  float* dpart = reinterpret_cast<float*>(smem + L.dpart);
  float* red = reinterpret_cast<float*>(smem + L.red);
  const int act_ld = 8 * L.max_groups;
  __half* act_s = act;
  __half* act_r = act + B * act_ld;

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
  stamp(1);

  // 1. router rows e = i, i + G, ... of this CTA (fp32 logits, all 8 warps
  //    split D), published to global memory + the launch's route counter
  {
    const int nch = D / 8;
    int rows = 0;
    if (L.rrows && i < E) mbar_wait(rrow_bar, 0);
    for (int e = i; e < E; e += G, ++rows) {
      const uint4* wr = reinterpret_cast<const uint4*>(p.w_router + (size_t)e * D);
      const uint4* ws = reinterpret_cast<const uint4*>(smem + L.rrow + (size_t)rows * D * 2);
      float a[QB];
#pragma unroll
      for (int b = 0; b < QB; ++b) a[b] = 0.f;
      for (int c = tid; c < nch; c += kConsumerThreads) {
        const uint4 wv = L.rrows ? ws[c] : __ldg(wr + c);
        const uint32_t q[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          if (b < B) {
            const uint4 xv = lds128(xs + (size_t)b * D + c * 8);
            const uint32_t xr[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) a[b] = fma_f16_hi(q[j], xr[j], fma_f16_lo(q[j], xr[j], a[b]));
          }
        }
      }
#pragma unroll
      for (int b = 0; b < QB; ++b) {
        if (b < B) {
          const float sw = warp_allsum(a[b]);
          if (lane == 0) red[b * kNumConsumerWarps + warp] = sw;
        }
      }
      consumer_sync();
      if (tid < B) {
        float v = 0.f;
        for (int w = 0; w < kNumConsumerWarps; ++w) v += red[tid * kNumConsumerWarps + w];
        p.logits[tid * E + e] = v;
      }
      consumer_sync();
    }
    if (rows && tid == 0) {
      __threadfence();
      atomicAdd(p.barrier + 1, (unsigned long long)rows);
    }
  }
  stamp(2);

  // 2. gate/up GEMV of one chunk, SwiGLU, fp16 activations into act_dst
  int cnt = 0;
  auto gate_up = [&](const Phase& P, int n_groups, __half* act_dst) {
    const int rows = 16 * n_groups;
    tiled_gemv_phase<__half, QB, true>(P, ring, warp, lane, tid, cnt, xs, D, B, rows, part,
                                       [&](int row, int b, float v) { gu[b * rows + row] = v; });
    consumer_sync();
    for (int t = tid; t < B * 8 * n_groups; t += kConsumerThreads) {
      const int b = t / (8 * n_groups), j = t % (8 * n_groups);  // f = 2*tile + e
      const int tl = j >> 1, e = j & 1;
      const float g = gu[b * rows + 4 * tl + e], uu = gu[b * rows + 4 * tl + 2 + e];
      act_dst[b * act_ld + j] = __float2half_rn(__fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), uu));
    }
    consumer_sync();
  };

  // 3. routing, all consumer threads: rank_b(e) = #{e' : l_e' > l_e or
  //    (l_e' == l_e and e' < e)}; row b selects e iff rank < K (ties toward
  //    the lower id) and e lands at top-k position rank.  The union of the
  //    rows' experts is compacted in ascending id; gw[b][slot] = row b's gate
  //    weight (softmax probability * scale) or 0.  No dynamically indexed
  //    register arrays anywhere: with 227 KB of shared memory there is little
  //    L1 left, and local memory would round-trip to L2.
  auto route = [&]() {
    int* s_idx = reinterpret_cast<int*>(smem + L.tk);
    float* s_w = reinterpret_cast<float*>(s_idx + B * K);
    float* st = red;  // [B][2] row max, row sum
    if (tid == 0) {
      const unsigned long long target = (epoch + 1ull) * (unsigned long long)E;
      while (ld_acquire_u64(p.barrier + 1) < target) __nanosleep(32);
    }
    consumer_sync();
    stamp(11);
    for (int t = tid; t < B * E; t += kConsumerThreads) lg[t] = __ldcg(p.logits + t);
    consumer_sync();
    stamp(12);
    if (warp < B) {  // row statistics: warp b
      const float* l = lg + warp * E;
      float m = -INFINITY;
      for (int e = lane; e < E; e += 32) m = fmaxf(m, l[e]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float sum = 0.f;
      for (int e = lane; e < E; e += 32) sum += expf(l[e] - m);
      sum = warp_allsum(sum);
      if (lane == 0) {
        st[2 * warp] = m;
        st[2 * warp + 1] = sum;
      }
    }
    consumer_sync();
    // ranks: 4 threads per (row, expert) pair, each comparing a quarter of the row
    for (int t0 = 0; t0 < 4 * B * E; t0 += kConsumerThreads) {
      const int t = t0 + tid;
      const bool valid = t < 4 * B * E;
      const int pr = valid ? t >> 2 : 0, qt = t & 3;
      const int b = pr / E, e = pr % E;
      const float* l = lg + b * E;
      const float v = l[e];
      int r = 0;
      for (int e2 = qt; e2 < E; e2 += 4) {
        const float o = l[e2];
        r += (o > v || (o == v && e2 < e)) ? 1 : 0;
      }
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      if (valid && qt == 0) {
        float w = -1.0f;  // marker: not selected by row b
        if (r < K) {
          w = __fmul_rn(__fdiv_rn(expf(v - st[2 * b]), st[2 * b + 1]), p.scale);
          s_idx[b * K + r] = e;
          s_w[b * K + r] = w;
        }
        lg[(B + b) * E + e] = w;
      }
    }
    consumer_sync();
    stamp(13);
    if (warp == 0) {
      int U = 0;
      for (int base = 0; base < E; base += 32) {
        const int e = base + lane;
        bool f = false;
        for (int b = 0; b < B; ++b) f |= e < E && lg[(B + b) * E + e] >= 0.f;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) {
          const int pos = U + __popc(bal & ((1u << lane) - 1u));
          slot_e[pos] = e;
          for (int b = 0; b < B; ++b) gw[b * L.umax + pos] = fmaxf(lg[(B + b) * E + e], 0.f);
        }
        U += __popc(bal);
      }
      if (lane == 0) slot_e[L.umax] = U;
      if (i == 0 && p.route_idx)
        for (int t = lane; t < B * K; t += 32) {
          p.route_idx[t] = s_idx[t];
          if (p.route_w) p.route_w[t] = s_w[t];
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(route_bar);  // release the expert list to the producer
    }
    consumer_sync();
  };

  // 4. split-K down projection: warp w owns column segment w % Q, lanes own
  //    fixed columns; fp16 weights x fp16 activations (FHFMA, exact products,
  //    fp32 sums) per expert segment, then scaled by the gate weight
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
  auto down = [&](const Phase& P, const __half* a_src, int g_off) {
    const int nch = Wd / 8;
    const unsigned short* a16 = reinterpret_cast<const unsigned short*>(a_src);
    consume_phase(P, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
      for (int uu = 0; uu < it.nunits; ++uu) {
        const int gl = (it.unit0 + uu) / Q + g_off;  // local group (segment = warp % Q)
        const char* blk = slot + (size_t)uu * blkB;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          uint32_t a2[QB];
#pragma unroll
          for (int b = 0; b < QB; ++b) {
            const uint32_t h = b < B ? a16[b * act_ld + 8 * gl + r] : 0u;
            a2[b] = h | (h << 16);
          }
#pragma unroll
          for (int j = 0; j < kCpl; ++j) {
            const int c = lane + 32 * j;
            if (c < nch) {
              const uint4 wv = lds128(blk + ((size_t)r * nch + c) * 16);
              const uint32_t wr[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
              for (int b = 0; b < QB; ++b)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  acc[b][j][2 * q] = fma_f16_lo(wr[q], a2[b], acc[b][j][2 * q]);
                  acc[b][j][2 * q + 1] = fma_f16_hi(wr[q], a2[b], acc[b][j][2 * q + 1]);
                }
            }
          }
        }
      }
    });
  };
  auto flush = [&](const float* wgt, bool add) {  // dpart[warp / Q][b][seg cols] (+)= w_b * acc
    float* dst = dpart + (size_t)(warp / Q) * B * D + (warp % Q) * Wd;
    const int nch = Wd / 8;
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      if (b < B) {
        const float w = wgt ? wgt[b * L.umax] : 1.0f;
#pragma unroll
        for (int j = 0; j < kCpl; ++j) {
          const int c = lane + 32 * j;
          if (c < nch) {
            float4* d4 = reinterpret_cast<float4*>(dst + (size_t)b * D + c * 8);
            float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (add) {
              const float4 o0 = d4[0], o1 = d4[1];
              o[0] = o0.x; o[1] = o0.y; o[2] = o0.z; o[3] = o0.w;
              o[4] = o1.x; o[5] = o1.y; o[6] = o1.z; o[7] = o1.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = fmaf(w, acc[b][j][e], o[e]);
            d4[0] = make_float4(o[0], o[1], o[2], o[3]);
            d4[1] = make_float4(o[4], o[5], o[6], o[7]);
          }
        }
      }
    }
  };

  // routing first (the producer streams the shared experts meanwhile and
  // needs the expert list before its ring is full), then shared gate/up and
  // down, routed gate/up and down
  route();
  stamp(3);
  // one schedule loop with a single call site per phase kind, so the large
  // unrolled gate/up and down bodies exist once in the binary (one-shot code
  // runs from a cold instruction cache every launch):
  //   pass 0 shared gate/up chunks, 1 shared down, 2 routed gate/up, 3 routed down
  const int U = slot_e[L.umax];
  const MoeRange m = moe_range(i, G, Gs, U * Ge);
  const int u_first = m.r0 / Ge;
  for (int pass = 0; pass < 4; ++pass) {
    const bool routed = pass >= 2, dn = pass & 1;
    const int nseg = routed ? max(0, min(U, (m.r1 + Ge - 1) / Ge) - u_first) : 1;
    for (int sg = 0; sg < nseg; ++sg) {
      int ga, gb, e = 0;
      const __half *gub, *dnb;
      __half* act_seg;
      int g_off;  // local group index = group index within the segment's matrix + g_off
      if (routed) {
        const int u = u_first + sg;
        e = seg(m, u, ga, gb);
        gub = p.w_gu + e * eGu;
        dnb = p.w_dn + e * eDn;
        act_seg = act_r;
        g_off = u * Ge - m.r0;
      } else {
        ga = rs.s0;
        gb = rs.s1;
        gub = p.s_gu;
        dnb = p.s_dn;
        act_seg = act_s;
        g_off = -rs.s0;
      }
      if (!dn) {
        for (int g = ga; g < gb; g += kMoeChunk)
          gate_up(gu_phase(gub, g, min(kMoeChunk, gb - g)), min(kMoeChunk, gb - g),
                  act_seg + 8 * (g + g_off));
      } else {
        zero_acc();
        down(dn_phase(dnb, ga, gb - ga), act_seg, ga + g_off);
        flush(routed ? gw + (u_first + sg) : nullptr, routed || sg > 0);
      }
    }
    if (pass == 1 && nseg == 0) {  // no shared experts: the routed flushes add onto zeros
      zero_acc();
      flush(nullptr, false);
    }
  }
  consumer_sync();
  stamp(7);

  // 5. this CTA's split-K partial -> its row of the partial buffer (plain
  //    coalesced stores, no atomics)
  const int nparts = 8 / Q, BD = B * D;
  for (int t = tid; t < BD; t += kConsumerThreads) {
    float v = 0.f;
    for (int s2 = 0; s2 < nparts; ++s2) v += dpart[(size_t)s2 * BD + t];
    p.part[(size_t)i * BD + t] = v;
  }
  stamp(8);
  // 6. barrier[0] (monotonic, G arrivals per launch; `epoch` read at launch):
  //    every CTA arrives; only the first NF CTAs wait and finish a column
  //    slice each, the others leave their SM to the next launch at once.
  //    out = [resid + attention sum +] sum over the G partial rows, summed as
  //    8 row-interleaved subsets (coalesced 32-column reads, all <= 20 loads
  //    of a thread in flight at once) combined in fixed order -
  //    deterministic, nothing to re-zero
  const int NF = G < 64 ? G : 64;
  consumer_sync();
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p.barrier) : "memory");
    if (i < NF) spin_until_geq(p.barrier, (epoch + 1ull) * (unsigned long long)G);
  }
  if (i >= NF) return;
  consumer_sync();
  stamp(9);
  const int c0 = (int)((long long)i * BD / NF), c1 = (int)((long long)(i + 1) * BD / NF);
  float* fsum = dpart;  // [8][32] row-subset sums
  const int ci = tid & 31, rg = tid >> 5;
  for (int cb = c0; cb < c1; cb += 32) {
    const int c = cb + ci;
    float acc = 0.f;
    if (c < c1) {
      constexpr int kRows = 20;  // G <= 160 rows / 8 subsets
      float v[kRows];
#pragma unroll
      for (int k = 0; k < kRows; ++k) v[k] = rg + 8 * k < G ? __ldcg(p.part + (size_t)(rg + 8 * k) * BD + c) : 0.f;
#pragma unroll
      for (int k = 0; k < kRows; ++k) acc += v[k];
    }
    fsum[rg * 32 + ci] = acc;
    consumer_sync();
    if (tid < 32 && cb + tid < c1) {
      const int cc = cb + tid;
      float v = 0.f;
#pragma unroll
      for (int g2 = 0; g2 < 8; ++g2) v += fsum[g2 * 32 + tid];
      float o = v;
      if (p.flags & CFB_RESID) {
        float r = __ldcg(p.resid + cc);
        if (p.accum_in) {
          r = __fadd_rn(r, fixed_to_float(__ldcg(p.accum_in + cc)));
          p.accum_in[cc] = 0ull;  // its norm readers (every CTA's prologue) are behind the barrier
        }
        if (!(p.flags & CFB_PARTIAL)) o = __fadd_rn(r, v);  // TP rank > 0: its expert-shard partial only
      }
      p.out[cc] = o;
    }
    consumer_sync();
  }
  stamp(10);
}

template <int QB>
static int launch_moe_inst(const MoeParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = moe_kernel<QB>;
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
  if (!a->w_router || !a->w_gu || !a->w_dn || (Fs && (!a->s_gu || !a->s_dn)) || !a->part ||
      !a->out || !a->barrier || !a->logits)
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
  if (grid > sms) grid = sms;         // routing waits on every CTA's router rows: co-resident
  if (grid > 160) grid = 160;         // the finalize holds <= 20 partial rows per thread
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
  p.part = a->part;
  p.out = a->out;
  p.route_idx = a->route_idx;
  p.route_w = a->route_w;
  p.barrier = a->barrier;
  p.trace = a->trace;
  p.logits = a->logits;
  const size_t smem = L.total;
  if (p.B == 1) return launch_moe_inst<1>(p, grid, smem, st);
  if (p.B == 2) return launch_moe_inst<2>(p, grid, smem, st);
  return launch_moe_inst<4>(p, grid, smem, st);
}

}  // namespace cfb
