// Persistent whole-step decode kernel (Llama2 family, batch 1): ONE launch
// per token runs embed -> n_layers x (attention module, SwiGLU FFN) -> LM
// head + argmax on every SM of the B200.
//
// Why: at batch 1 a decode step is a pure HBM stream (13.2 GB of weights per
// token, 1 flop/byte).  The layered engine (csrc/llama.cu) loses ~20 % of the
// roofline at kernel boundaries: each launch starts with an empty ring once
// the previous launch's last CTA has left, and the split_token attention
// module runs on 128 of the 148 SMs (32 heads x cluster 4).  Here every CTA's
// producer warp streams its share of ALL layers' weights and KV rows without
// ever stopping - weights never depend on activations - and the consumers
// synchronise through global-memory flags only where the dataflow has a real
// dependency.  While consumers wait, the producer keeps filling the 192 KB
// ring with the next phase's bytes (~4 us of this SM's HBM share), so a wait
// shorter than that costs no bandwidth.
//
// Work per layer, per CTA i of G (static, contiguous, balanced ranges):
//   A. RMSNorm(resid) -> QKV GEMV over tiles [i*TQ/G, (i+1)*TQ/G) of the
//      split_token W_qkv layout (the same packed weights as the cluster
//      kernel), q|k|v rows fp16-stored to a global buffer; per-head counter
//      qkv_done[h] += tiles of head h done here.
//   B. split-KV flash decoding (reference dataflows.py:71-99 partial
//      attention, :109-114 contiguous segments) over the flattened
//      (head, position) space [0, nh*(S+1)): CTA i's range is one or two
//      head pieces; a piece waits for its head's q/k/v, applies RoPE, appends
//      the new K/V row (the CTA owning position S), attends its rows (the new
//      token's K/V counted once, by the piece that holds position S - SPEC.md:284)
//      and writes an fp32 partial (m, l, A) to global memory; att_done[h]++.
//   C. O projection over the flattened (head, output column) rows: per head
//      in range, wait for all pieces of the head, merge them (the
//      reference's max-reduce / rescale / sum-reduce / rescale,
//      dataflows.py:187-232, in fp32, fixed order), round A to fp16 and run
//      the row-per-lane GEMV; outputs go to the 64-bit fixed-point head-sum
//      accumulator (red.add: exact, order-free) - reference
//      atomic_accumulate, dataflows.py:302-310.
//   -- grid barrier --
//   D. RMSNorm(resid + accum) -> gate/up GEMV -> SiLU*mul -> act (fp16, global)
//   -- grid barrier --
//   E. down GEMV over rows [i*D/4/G ..) -> resid = resid + accum + ffn; accum = 0
//   -- grid barrier --
// then RMSNorm + LM head + argmax (ticketed last CTA writes the token and
// advances the position).  The attention here exchanges partials through
// global memory (L2) instead of DSMEM: a flattened split over all SMs does
// not map onto fixed clusters; the cluster dataflow stays in
// csrc/attn_mha.cu (drop-in API and layered engine).
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

namespace {

constexpr int kH = 128;         // head dim (Llama family)
constexpr int kEPL = 16;        // attention elements per lane
constexpr int kLPK = kH / kEPL; // lanes per key (8)
constexpr int kKPP = 32 / kLPK; // keys per warp step (4)
constexpr int kRC = 4;          // warp steps per online-softmax chunk
constexpr int kPS = kH + 4;     // floats per attention partial: m, l, pad, pad, A[H]

struct StepParams {
  int L, D, nh, F, V, cap, N, tpr, spw, sleep_max;
  float eps, inv_sqrt_h;
  const __half* const* attn_norm;
  const __half* const* w_qkv;
  const __half* const* w_out;
  const __half* const* ffn_norm;
  const __half* const* w_gu;
  const __half* const* w_dn;
  __half* const* k_cache;
  __half* const* v_cache;
  const __half* embed;
  const __half* final_norm;
  const __half* lm_head;
  const float* rope_cs;
  float* resid;                  // [D] fp32 residual stream
  unsigned long long* accum;     // [D] fixed-point head sum
  __half* qkv;                   // [nh * N * tpr * 4] q|k|v rows of the layer
  __half* act;                   // [F]
  float* partials;               // [nh][G][kPS]
  unsigned long long* barrier;   // grid barrier counter (monotonic)
  unsigned long long* counters;  // [2 * nh]: qkv_done, att_done (zeroed per step)
  float* logits;                 // [V]
  float* cand_val;               // [G]
  int* cand_idx;                 // [G]
  unsigned* ticket;
  int* token;
  int* pos;
  int* err;                      // set to 1 when pos + 1 > cache capacity (step skipped)
  unsigned long long* trace;     // [L][G][8] globaltimer stamps (nullable)
};

struct StepLayout {
  int bars, xs, part, gu, qf, red, misc, total, max_rows;
};

__host__ __device__ inline int r16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline StepLayout step_layout(int D, int F, int TQ, int TV, int G, int spw) {
  StepLayout L;
  auto tiles = [&](int T) { return (T + G - 1) / G; };
  int t = tiles(TQ);
  if (tiles(F / 2) > t) t = tiles(F / 2);
  if (tiles(D / 4) > t) t = tiles(D / 4);
  if (tiles(TV) > t) t = tiles(TV);
  L.max_rows = 4 * t;
  int part = kNumConsumerWarps * L.max_rows * 4;
  const int ws = kNumConsumerWarps * kPS * 4;  // attention warp states alias `part`
  if (ws > part) part = ws;
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.xs = o;    o += r16((D > F ? D : F) * 2);
  L.part = o;  o += r16(part);
  L.gu = o;    o += r16(4 * tiles(F / 2) * 4);
  L.qf = o;    o += 3 * kH * 4 + kH * 2;  // q, k, v fp32 + fp16 A for the O projection
  L.red = o;   o += r16(kNumConsumerWarps * 4 * 2);
  L.misc = o;  o += 64;
  L.total = o;
  return L;
}

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

__device__ __forceinline__ long long split_at(long long total, int i, int G) {
  return total * i / G;
}

// CTA owning flat position x of a [0, total) split into G contiguous ranges
__device__ __forceinline__ int owner_of(long long x, long long total, int G) {
  const long long i = ((x + 1) * G - 1) / total;
  return (int)(i < G - 1 ? i : G - 1);
}

__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// thread 0 spins until *p >= target, then the CTA's consumers proceed
__device__ __forceinline__ void wait_counter(const unsigned long long* p, unsigned long long target,
                                             int tid) {
  if (tid == 0) {
    while (ld_acquire_u64(p) < target) __nanosleep(32);
    __threadfence();
  }
  consumer_sync();
}

// One chunked online-softmax pass of a warp over `nkeys` K/V rows (row
// stride kH) - the same per-lane arithmetic as the split_token kernel.
template <class LoadK, class LoadV>
__device__ __forceinline__ void attend(const float (&q)[kEPL], float& m, float& l,
                                       float (&acc)[kEPL], int nkeys, int g, float scale,
                                       LoadK&& load_k, LoadV&& load_v) {
  for (int k0 = 0; k0 < nkeys; k0 += kRC * kKPP) {
    float s[kRC];
    bool valid[kRC];
#pragma unroll
    for (int j = 0; j < kRC; ++j) {
      const int key = k0 + j * kKPP + g;
      valid[j] = key < nkeys;
      float kv[kEPL];
      load_k(valid[j] ? key : 0, kv);
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < kEPL; ++e) t = fmaf(q[e], kv[e], t);
      s[j] = t;
    }
#pragma unroll
    for (int o = 1; o < kLPK; o <<= 1)
#pragma unroll
      for (int j = 0; j < kRC; ++j) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    float vv[kRC][kEPL];
#pragma unroll
    for (int j = 0; j < kRC; ++j) load_v(valid[j] ? k0 + j * kKPP + g : 0, vv[j]);
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kRC; ++j) {
      s[j] = valid[j] ? __fmul_rn(s[j], scale) : -INFINITY;
      mx = fmaxf(mx, s[j]);
    }
#pragma unroll
    for (int o = kLPK; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float mn = fmaxf(m, mx);
    const float alpha = __expf(m - mn);
    float ps = 0.f;
#pragma unroll
    for (int e = 0; e < kEPL; ++e) acc[e] *= alpha;
#pragma unroll
    for (int j = 0; j < kRC; ++j) {
      const float pr = __expf(s[j] - mn);
      ps += pr;
#pragma unroll
      for (int e = 0; e < kEPL; ++e) acc[e] = fmaf(pr, vv[j][e], acc[e]);
    }
    l = fmaf(l, alpha, ps);
    m = mn;
  }
}

__device__ __forceinline__ void stamp(unsigned long long* tr, int k, int tid) {
  if (tr && tid == 0) tr[k] = globaltimer();
}

__global__ void __launch_bounds__(kThreads, 1) llama_step_kernel(const StepParams p) {
  extern __shared__ __align__(128) char smem[];
  const int G = gridDim.x, i = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = p.D, F = p.F, nh = p.nh, N = p.N;
  const int hp = kH / N;                      // head dims per split_token rank
  const int TPH = N * p.tpr;                  // W_qkv tiles per head
  const int TQ = nh * TPH, T1 = F / 2, T2 = D / 4, TV = p.V / 4;
  const StepLayout Lo = step_layout(D, F, TQ, TV, G, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lo.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};

  const int S = *p.pos;
  if (S + 1 > p.cap) {  // uniform across the grid: no barrier is entered
    if (i == 0 && tid == 0) *p.err = 1;
    return;
  }
  const long long SP = S + 1;                 // attended positions per head
  const long long PK = (long long)nh * SP;    // flattened (head, position) space
  const long long RO = (long long)nh * D;     // flattened (head, output column) rows

  // static ranges of this CTA
  const int q0 = (int)split_at(TQ, i, G), q1 = (int)split_at(TQ, i + 1, G);
  const long long k0 = split_at(PK, i, G), k1 = split_at(PK, i + 1, G);
  const long long o0 = split_at(RO, i, G), o1 = split_at(RO, i + 1, G);
  const int a0 = (int)split_at(T1, i, G), a1 = (int)split_at(T1, i + 1, G);
  const int u0 = (int)split_at(T2, i, G), u1 = (int)split_at(T2, i + 1, G);
  const int v0 = (int)split_at(TV, i, G), v1 = (int)split_at(TV, i + 1, G);
  // attention pieces: (head, [lo, hi) local positions), at most two
  int ph[2] = {0, 0}, plo[2] = {0, 0}, phi[2] = {0, 0}, npiece = 0;
  for (long long x = k0; x < k1 && npiece < 2;) {
    const int h = (int)(x / SP);
    const long long e = k1 < (h + 1) * SP ? k1 : (h + 1) * SP;
    ph[npiece] = h;
    plo[npiece] = (int)(x - h * SP);
    phi[npiece] = (int)(e - h * SP);
    ++npiece;
    x = e;
  }
  // O-projection pieces: (head, [c_lo, c_hi) output columns), at most two
  int oh[2] = {0, 0}, olo[2] = {0, 0}, ohi[2] = {0, 0}, nopiece = 0;
  for (long long x = o0; x < o1 && nopiece < 2;) {
    const int h = (int)(x / D);
    const long long e = o1 < (long long)(h + 1) * D ? o1 : (long long)(h + 1) * D;
    oh[nopiece] = h;
    olo[nopiece] = (int)(x - (long long)h * D);
    ohi[nopiece] = (int)(e - (long long)h * D);
    ++nopiece;
    x = e;
  }

  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();

  auto layer_phases = [&](int l, Phase (&P)[7]) {
    P[0] = make_phase(p.w_qkv[l] + (size_t)q0 * 4 * D, nullptr, q1 - q0, 4 * D * 2, true);
    for (int j = 0; j < 2; ++j) {
      const int n = j < npiece ? (phi[j] < S ? phi[j] : S) - plo[j] : 0;
      const size_t off = ((size_t)ph[j] * p.cap + (j < npiece ? plo[j] : 0)) * kH;
      P[1 + j] = make_phase(p.k_cache[l] + off, p.v_cache[l] + off, n > 0 ? n : 0, kH * 2);
    }
    for (int j = 0; j < 2; ++j) {
      // W_out rows of head oh[j], columns [olo, ohi): layout [head][rank][cols][H]
      // flattens to [head][column][H]
      const size_t off = ((size_t)oh[j] * D + (j < nopiece ? olo[j] : 0)) * kH;
      P[3 + j] = make_phase(p.w_out[l] + off, nullptr, j < nopiece ? ohi[j] - olo[j] : 0, kH * 2);
    }
    P[5] = make_phase(p.w_gu[l] + (size_t)a0 * 4 * D, nullptr, a1 - a0, 4 * D * 2, true);
    P[6] = make_phase(p.w_dn[l] + (size_t)u0 * 4 * F, nullptr, u1 - u0, 4 * F * 2, true);
  };

  if (warp == kNumConsumerWarps) {  // ---------------------------- producer
    const uint64_t pol = policy_evict_first();
    int c = 0;
    for (int l = 0; l < p.L; ++l) {
      Phase P[7];
      layer_phases(l, P);
      produce_all(P, ring, lane, pol, c);
    }
    const Phase PL[1] = {make_phase(p.lm_head + (size_t)v0 * 4 * D, nullptr, v1 - v0, 4 * D * 2, true)};
    produce_all(PL, ring, lane, pol, c);
    return;
  }

  // ------------------------------------------------------------------ consumers
  __half* xs = reinterpret_cast<__half*>(smem + Lo.xs);
  float* part = reinterpret_cast<float*>(smem + Lo.part);
  float* gu = reinterpret_cast<float*>(smem + Lo.gu);
  float* qf = reinterpret_cast<float*>(smem + Lo.qf);
  float* kf = qf + kH;
  float* vf = kf + kH;
  __half* abuf = reinterpret_cast<__half*>(vf + kH);
  float* red = reinterpret_cast<float*>(smem + Lo.red);
  unsigned* last = reinterpret_cast<unsigned*>(smem + Lo.misc);
  unsigned long long* qkv_done = p.counters;
  unsigned long long* att_done = p.counters + nh;

  // embed: resid[c] = embed[token][c] for this CTA's slice; counters reset
  {
    const int tok = *p.token;
    const int c0 = (int)split_at(D, i, G), c1 = (int)split_at(D, i + 1, G);
    for (int c = c0 + tid; c < c1; c += kConsumerThreads)
      p.resid[c] = __half2float(p.embed[(size_t)tok * D + c]);
    if (i == 0 && tid < 2 * nh) p.counters[tid] = 0ull;
  }
  grid_barrier(p.barrier, tid);

  // cross-CTA data is read through L2 (ld.global.cg): L1 is not coherent
  const float* resid_g = p.resid;
  auto resid_l2 = [resid_g](int, int v) { return __ldcg(reinterpret_cast<const float4*>(resid_g) + v); };
  int cnt = 0;
  const int rowsQ = 4 * (q1 - q0);
  const int g = lane / kLPK, li = lane % kLPK;
  const float scale = p.inv_sqrt_h;
  const int half = kH / 2;
  for (int l = 0; l < p.L; ++l) {
    unsigned long long* tr = p.trace ? p.trace + ((size_t)l * G + i) * 8 : nullptr;
    stamp(tr, 0, tid);
    Phase P[7];
    layer_phases(l, P);
    // ---- A. QKV projection
    rmsnorm_to_smem_ld<__half, true>(xs, resid_l2, p.attn_norm[l], 1, D, p.eps, red, tid);
    tiled_gemv_phase<__half, 1, true>(P[0], ring, warp, lane, tid, cnt, xs, D, 1, rowsQ, part,
                                      [&](int row, int, float v) {
                                        p.qkv[(size_t)4 * q0 + row] = __float2half_rn(v);
                                      });
    __threadfence();
    consumer_sync();
    if (tid == 0) {
      for (int h = q0 / TPH; h < nh && h * TPH < q1; ++h) {
        const int lo = max(q0, h * TPH), hi = min(q1, (h + 1) * TPH);
        red_release_add(&qkv_done[h], (unsigned long long)(hi - lo));
      }
    }
    stamp(tr, 1, tid);

    // ---- B. attention pieces
    for (int j = 0; j < 2; ++j) {
      const Phase& PK_ = P[1 + j];
      if (j >= npiece) {  // keep the ring walk aligned (phase is empty)
        continue;
      }
      const int h = ph[j];
      const bool has_new = phi[j] == S + 1;
      wait_counter(&qkv_done[h], (unsigned long long)TPH * (l + 1), tid);
      // q, k_new, v_new of head h from the split_token row order
      for (int d = tid; d < kH; d += kConsumerThreads) {
        const size_t r = ((size_t)h * N + d / hp) * p.tpr * 4 + d % hp;
        qf[d] = __half2float(__ldcg(p.qkv + r));
        kf[d] = __half2float(__ldcg(p.qkv + r + hp));
        vf[d] = __half2float(__ldcg(p.qkv + r + 2 * hp));
      }
      consumer_sync();
      for (int d = tid; d < half; d += kConsumerThreads) {  // RoPE at position S
        const float c = p.rope_cs[((size_t)S * half + d) * 2];
        const float sn = p.rope_cs[((size_t)S * half + d) * 2 + 1];
        const float q1_ = qf[d], q2 = qf[d + half], k1_ = kf[d], k2 = kf[d + half];
        qf[d] = round_to<__half>(__fsub_rn(__fmul_rn(q1_, c), __fmul_rn(q2, sn)));
        qf[d + half] = round_to<__half>(__fadd_rn(__fmul_rn(q2, c), __fmul_rn(q1_, sn)));
        kf[d] = round_to<__half>(__fsub_rn(__fmul_rn(k1_, c), __fmul_rn(k2, sn)));
        kf[d + half] = round_to<__half>(__fadd_rn(__fmul_rn(k2, c), __fmul_rn(k1_, sn)));
      }
      consumer_sync();
      if (has_new) {  // KV-cache append at row S (read by later steps only)
        const size_t off = ((size_t)h * p.cap + S) * kH;
        for (int d = tid; d < kH; d += kConsumerThreads) {
          p.k_cache[l][off + d] = __float2half_rn(kf[d]);
          p.v_cache[l][off + d] = __float2half_rn(vf[d]);
        }
      }
      float q[kEPL], acc[kEPL], m = -INFINITY, lsum = 0.f;
#pragma unroll
      for (int e = 0; e < kEPL; ++e) {
        q[e] = qf[li * kEPL + e];
        acc[e] = 0.f;
      }
      consume_phase(PK_, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
        const __half* K = reinterpret_cast<const __half*>(slot);
        const __half* V = reinterpret_cast<const __half*>(slot + kSlotBytes / 2);
        attend(q, m, lsum, acc, it.nunits, g, scale,
               [&](int k, float* o) { load_elems<__half, kEPL>(K + k * kH + li * kEPL, o); },
               [&](int k, float* o) { load_elems<__half, kEPL>(V + k * kH + li * kEPL, o); });
      });
      if (has_new && warp == 0)
        attend(q, m, lsum, acc, 1, g, scale,
               [&](int, float* o) {
#pragma unroll
                 for (int e = 0; e < kEPL; ++e) o[e] = kf[li * kEPL + e];
               },
               [&](int, float* o) {
#pragma unroll
                 for (int e = 0; e < kEPL; ++e) o[e] = vf[li * kEPL + e];
               });
      // fold the key groups of the warp (same dims), then the 8 warps in order
#pragma unroll
      for (int o = kLPK; o < 32; o <<= 1) {
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
#pragma unroll
        for (int e = 0; e < kEPL; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
      }
      float* ws = part + warp * kPS;
      if (g == 0) {
#pragma unroll
        for (int e = 0; e < kEPL; ++e) ws[4 + li * kEPL + e] = acc[e];
      }
      if (lane == 0) {
        ws[0] = m;
        ws[1] = lsum;
      }
      consumer_sync();
      float* dst = p.partials + ((size_t)h * G + i) * kPS;
      for (int d = tid; d < kH; d += kConsumerThreads) {
        float mm = -INFINITY;
#pragma unroll
        for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) mm = fmaxf(mm, part[w2 * kPS]);
        float ll = 0.f, a = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) {
          const float mw = part[w2 * kPS];
          const float f = (mw == -INFINITY) ? 0.f : expf(mw - mm);
          ll = fmaf(part[w2 * kPS + 1], f, ll);
          a = fmaf(part[w2 * kPS + 4 + d], f, a);
        }
        dst[4 + d] = a;
        if (d == 0) {
          dst[0] = mm;
          dst[1] = ll;
        }
      }
      __threadfence();
      consumer_sync();
      if (tid == 0) red_release_add(&att_done[h], 1ull);
    }
    stamp(tr, 2, tid);

    // ---- C. merge + O projection into the fixed-point head sum
    for (int j = 0; j < nopiece; ++j) {
      const int h = oh[j];
      const long long ha = (long long)h * SP, hb = ha + SP;
      const int first = owner_of(ha, PK, G), lastc = owner_of(hb - 1, PK, G);
      int npieces = 0;
      for (int c = first; c <= lastc; ++c)
        npieces += split_at(PK, c, G) < split_at(PK, c + 1, G);
      wait_counter(&att_done[h], (unsigned long long)npieces * (l + 1), tid);
      for (int d = tid; d < kH; d += kConsumerThreads) {
        float ms = -INFINITY;
        for (int c = first; c <= lastc; ++c)
          if (split_at(PK, c, G) < split_at(PK, c + 1, G))
            ms = fmaxf(ms, __ldcg(p.partials + ((size_t)h * G + c) * kPS));
        float ls = 0.f, a = 0.f;
        for (int c = first; c <= lastc; ++c) {
          if (split_at(PK, c, G) >= split_at(PK, c + 1, G)) continue;
          const float* src = p.partials + ((size_t)h * G + c) * kPS;
          const float mr = __ldcg(src);
          const float f = (mr == -INFINITY) ? 0.f : expf(mr - ms);
          ls = fmaf(__ldcg(src + 1), f, ls);
          a = fmaf(__ldcg(src + 4 + d), f, a);
        }
        abuf[d] = __float2half_rn(__fdiv_rn(a, ls));
      }
      consumer_sync();
      const int c_lo = olo[j];
      consume_phase(P[3 + j], ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
        // absolute column index: the packed rows are chunk-rotated by their row
        // within the rank slice, (c mod D/N) mod 16 == c mod 16 (host-checked)
        Item it2 = it;
        it2.unit0 += c_lo;
        rowlane_item<__half, 1>(it2, slot, abuf, kH, 1, lane, [&](int col, const float (&s)[1]) {
          red_add_fixed(&p.accum[col], s[0]);
        });
      });
    }
    stamp(tr, 3, tid);
    grid_barrier(p.barrier, tid);
    stamp(tr, 4, tid);

    // ---- D. FFN gate/up with the residual + head-sum RMSNorm prologue
    {
      const float* resid = p.resid;
      const unsigned long long* acc = p.accum;
      rmsnorm_to_smem_ld<__half, true>(
          xs,
          [&](int, int v) {
            const float4 r = __ldcg(reinterpret_cast<const float4*>(resid) + v);
            const ulonglong2 x0 = __ldcg(reinterpret_cast<const ulonglong2*>(acc) + 2 * v);
            const ulonglong2 x1 = __ldcg(reinterpret_cast<const ulonglong2*>(acc) + 2 * v + 1);
            return make_float4(__fadd_rn(r.x, fixed_to_float(x0.x)), __fadd_rn(r.y, fixed_to_float(x0.y)),
                               __fadd_rn(r.z, fixed_to_float(x1.x)), __fadd_rn(r.w, fixed_to_float(x1.y)));
          },
          p.ffn_norm[l], 1, D, p.eps, red, tid);
    }
    const int rows0 = 4 * (a1 - a0);
    tiled_gemv_phase<__half, 1, true>(P[5], ring, warp, lane, tid, cnt, xs, D, 1, rows0, part,
                                      [&](int row, int, float v) { gu[row] = v; });
    consumer_sync();
    for (int jj = tid; jj < 2 * (a1 - a0); jj += kConsumerThreads) {
      const int t = jj >> 1, e = jj & 1;  // tile rows: g0 g1 u0 u1
      const float gt = gu[4 * t + e], up = gu[4 * t + 2 + e];
      const float sl = __fdiv_rn(gt, __fadd_rn(1.0f, expf(-gt)));
      p.act[2 * a0 + jj] = __float2half_rn(__fmul_rn(sl, up));
    }
    stamp(tr, 5, tid);
    grid_barrier(p.barrier, tid);
    stamp(tr, 6, tid);

    // ---- E. down projection + residual
    load_act_to_smem<__half, true>(xs, p.act, 1, F, tid);
    tiled_gemv_phase<__half, 1, true>(P[6], ring, warp, lane, tid, cnt, xs, F, 1, 4 * (u1 - u0), part,
                                      [&](int row, int, float v) {
                                        const int c = 4 * u0 + row;
                                        const float r = __fadd_rn(__ldcg(p.resid + c),
                                                                  fixed_to_float(__ldcg(p.accum + c)));
                                        p.accum[c] = 0ull;
                                        p.resid[c] = __fadd_rn(r, v);
                                      });
    stamp(tr, 7, tid);
    grid_barrier(p.barrier, tid);
  }

  // ---- final RMSNorm + LM head + argmax
  rmsnorm_to_smem_ld<__half, true>(xs, resid_l2, p.final_norm, 1, D, p.eps, red, tid);
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  const Phase PL = make_phase(p.lm_head + (size_t)v0 * 4 * D, nullptr, v1 - v0, 4 * D * 2, true);
  tiled_gemv_phase<__half, 1, true>(PL, ring, warp, lane, tid, cnt, xs, D, 1, 4 * (v1 - v0), part,
                                    [&](int row, int, float s) {
                                      const int v = 4 * v0 + row;
                                      if (v >= p.V) return;
                                      p.logits[v] = s;
                                      if (better(s, v, bv, bi)) {
                                        bv = s;
                                        bi = v;
                                      }
                                    });
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    red[warp] = bv;
    reinterpret_cast<int*>(red)[kNumConsumerWarps + warp] = bi;
  }
  consumer_sync();
  if (tid == 0) {
    float v = -INFINITY;
    int ix = 0x7fffffff;
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2)
      if (better(red[w2], reinterpret_cast<int*>(red)[kNumConsumerWarps + w2], v, ix)) {
        v = red[w2];
        ix = reinterpret_cast<int*>(red)[kNumConsumerWarps + w2];
      }
    p.cand_val[i] = v;
    p.cand_idx[i] = ix;
    __threadfence();
    *last = (atomicAdd(p.ticket, 1u) == (unsigned)G - 1);
  }
  consumer_sync();
  if (*last && tid == 0) {
    __threadfence();
    float v = -INFINITY;
    int ix = 0x7fffffff;
    for (int c = 0; c < G; ++c) {
      const float cv = __ldcg(&p.cand_val[c]);
      const int ci = __ldcg(&p.cand_idx[c]);
      if (better(cv, ci, v, ix)) {
        v = cv;
        ix = ci;
      }
    }
    *p.token = ix;
    *p.ticket = 0;
    *p.pos = S + 1;
  }
}

}  // namespace

int llama_step_smem(int D, int F, int nh, int N, int tpr, int V, int G, int* spw_out) {
  int spw = tuned_spw();
  const int TQ = nh * N * tpr, TV = V / 4;
  StepLayout L = step_layout(D, F, TQ, TV, G, spw);
  while (L.total > kMaxSmem && spw > 1) L = step_layout(D, F, TQ, TV, G, --spw);
  if (spw_out) *spw_out = spw;
  return L.total;
}

int llama_step_launch(const LlamaStepArgs* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->head_dim != kH) return set_error(CFB_ERR_DIMENSION, "persistent engine needs head_dim 128");
  const int N = a->cluster;
  if (N < 1 || N > 16 || (N & (N - 1)) || kH % N)
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16]");
  if (a->hidden % 8 || a->inter % 8 || a->vocab % 4 || (a->hidden / N) % (kH * 2 / 16))
    return set_error(CFB_ERR_DIMENSION, "persistent engine: hidden/inter multiples of 8, vocab of 4");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int G = a->grid > 0 && a->grid < sms ? a->grid : sms;
  if (G < a->n_heads)  // a CTA's flattened ranges then span at most two heads
    return set_error(CFB_ERR_DIMENSION, "persistent engine: grid %d vs %d heads", G, a->n_heads);
  int spw = 0;
  const int tpr = (3 * (kH / N) + 3) / 4;
  const int smem = llama_step_smem(a->hidden, a->inter, a->n_heads, N, tpr, a->vocab, G, &spw);
  if (smem > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "persistent engine needs %d B of shared memory (max %d)", smem,
                     kMaxSmem);
  StepParams p;
  p.L = a->n_layers;
  p.D = a->hidden;
  p.nh = a->n_heads;
  p.F = a->inter;
  p.V = a->vocab;
  p.cap = a->cache_cap;
  p.N = N;
  p.tpr = tpr;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.eps = a->eps;
  p.inv_sqrt_h = (float)(1.0 / std::sqrt((double)kH));
  p.attn_norm = reinterpret_cast<const __half* const*>(a->attn_norm);
  p.w_qkv = reinterpret_cast<const __half* const*>(a->w_qkv);
  p.w_out = reinterpret_cast<const __half* const*>(a->w_out);
  p.ffn_norm = reinterpret_cast<const __half* const*>(a->ffn_norm);
  p.w_gu = reinterpret_cast<const __half* const*>(a->w_gu);
  p.w_dn = reinterpret_cast<const __half* const*>(a->w_dn);
  p.k_cache = reinterpret_cast<__half* const*>(a->k_cache);
  p.v_cache = reinterpret_cast<__half* const*>(a->v_cache);
  p.embed = static_cast<const __half*>(a->embed);
  p.final_norm = static_cast<const __half*>(a->final_norm);
  p.lm_head = static_cast<const __half*>(a->lm_head);
  p.rope_cs = a->rope_cs;
  p.resid = a->resid;
  p.accum = a->accum;
  p.qkv = static_cast<__half*>(a->qkv);
  p.act = static_cast<__half*>(a->act);
  p.partials = a->partials;
  p.barrier = a->barrier;
  p.counters = a->counters;
  p.logits = a->logits;
  p.cand_val = a->cand_val;
  p.cand_idx = a->cand_idx;
  p.ticket = a->ticket;
  p.token = a->token;
  p.pos = a->pos;
  p.err = a->err;
  p.trace = a->trace;
  auto kern = llama_step_kernel;
  CFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

}  // namespace cfb
