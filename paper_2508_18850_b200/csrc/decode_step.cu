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

#include "collectives.cuh"
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
  const int* kv_pages;           // paged KV: block table [cap / 128] (page ids, -1 = none), or null;
                                 // the caches are then page pools: row r of head h at element
                                 // h * kv_hstride + pages[r / 128] * kv_pstride + (r % 128) * H
  long long kv_pstride, kv_hstride;
  const __half* embed;
  const __half* final_norm;
  const __half* lm_head;
  const float* rope_cs;
  float* resid;                  // [D] fp32 residual stream
  unsigned long long* accA;      // [D] fixed-point attention head sum
  __half* act;                   // [F] SwiGLU activations
  __half* qkv;                   // [nh * N * tpr * 4] q|k|v rows of the layer
  float* partials;               // [nh][G][kPS]
  unsigned long long* barrier;   // grid barrier counter (monotonic)
  unsigned long long* counters;  // [2 * nh]: qkv_done, att_done (zeroed per step)
  unsigned long long* pool_ctr;  // [L] gate/up work-stealing counters (monotonic)
  int pool;                      // gate/up tiles per layer handed out dynamically
  float* logits;                 // [V]
  float* cand_val;               // [G]
  int* cand_idx;                 // [G]
  unsigned* ticket;
  int* token;
  int* pos;
  int* err;                      // set to 1 when pos + 1 > cache capacity (step skipped)
  unsigned long long* trace;     // [L][G][8] globaltimer stamps (nullable)
  // tensor parallel (T > 1): see tp_* below
  int T, trank, voff;
  unsigned long long* const* xch;  // [T] exchange blocks (peer-mapped)
  float* resid2;
  unsigned long long* uc_sum;  // NVLS: this rank's copy of the sums [6][D] (else null)
  unsigned long long* mc_sum;  // NVLS: multicast mapping of the same buffer
  long long timeout_ns;
  int l2_prefetch;               // bytes per CTA prefetched into L2 past the ring at each barrier
};

// ---------------------------------------------------------------- tensor parallel
// Rank r holds heads [r nh/T ..), FFN columns [r F/T ..) and LM-head rows
// [r V/T ..) (Megatron), so each block half ends in a SUM all-reduce of a
// D-vector.  Here the all-reduce is part of the kernel: every CTA owns a
// D/G slice and red.adds it, as 64-bit fixed point (exact, order-free: the
// sum is bit-identical whatever the arrival order), straight into every
// rank's exchange block over NVLink peer memory, then the T x G CTAs meet at
// a cross-rank counter (red.release.sys / ld.acquire.sys).  Exchange block
// of a rank (u64 words): XA [3][D] attention sums, XF [3][D] FFN sums, then
// the barrier counter, argmax key and token counter on separate lines.
// Layer l uses set l % 3 and residual buffer l & 1; layer l zeroes its slice
// of set (l + 1) % 3, whose last reader (layer l - 1) is behind the previous
// cross barrier and whose next writers (layer l + 1) are behind the next one.
__device__ __forceinline__ unsigned long long* tp_xa(unsigned long long* x, int D, int s) {
  return x + (size_t)s * D;
}
__device__ __forceinline__ unsigned long long* tp_xf(unsigned long long* x, int D, int s) {
  return x + (size_t)(3 + s) * D;
}
__device__ __forceinline__ unsigned long long* tp_bar(unsigned long long* x, int D) { return x + 6 * (size_t)D; }
__device__ __forceinline__ unsigned long long* tp_key(unsigned long long* x, int D) { return x + 6 * (size_t)D + 16; }
__device__ __forceinline__ unsigned long long* tp_tok(unsigned long long* x, int D) { return x + 6 * (size_t)D + 32; }

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// NVLS: one reduction on the multicast address updates every rank's copy
__device__ __forceinline__ void multimem_red_add_u64(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
// this slice element of the layer's sum to every rank: one multicast
// reduction (NVLS) or one peer-memory reduction per rank
__device__ __forceinline__ void tp_push(const StepParams& p, int set, int c, unsigned long long v) {
  if (p.mc_sum) {
    multimem_red_add_u64(p.mc_sum + (size_t)set * p.D + c, v);
  } else {
    for (int t = 0; t < p.T; ++t) red_add_u64(p.xch[t] + (size_t)set * p.D + c, v);
  }
}

// spin (thread 0) until *ctr >= target; on expiry of the bound set err = 2
// and give up (the step's result is then garbage, but nothing hangs)
__device__ __forceinline__ void tp_spin(const unsigned long long* ctr, unsigned long long target,
                                        long long timeout_ns, int* err) {
  unsigned long long t0 = 0;
  while (ld_acquire_sys_u64(ctr) < target) {
    if (timeout_ns > 0) {
      const unsigned long long t = globaltimer();
      if (!t0) {
        t0 = t;
      } else if ((long long)(t - t0) > timeout_ns) {
        atomicExch(err, 2);
        break;
      }
    }
  }
}

// all T x G CTAs of the tensor-parallel group meet (target = base + k T G)
__device__ __forceinline__ void cross_sync(const StepParams& p, unsigned long long target, int tid) {
  consumer_sync();
  if (tid == 0) {
    __threadfence_system();  // cumulative over the CTA's writes ordered by the bar.sync above
    for (int t = 0; t < p.T; ++t) red_release_sys_add(tp_bar(p.xch[t], p.D), 1ull);
    tp_spin(tp_bar(p.xch[p.trank], p.D), target, p.timeout_ns, p.err);
    __threadfence();
  }
  consumer_sync();
}

// order-preserving key: larger logit wins, equal logits -> smaller index
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  const unsigned u = __float_as_uint(v);
  const unsigned o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | (unsigned long long)(0xFFFFFFFFu - (unsigned)idx);
}

struct StepLayout {
  int bars, xs, part, gu, qf, dsm, red, tag, misc, total, max_rows;
};

__host__ __device__ inline int r16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline StepLayout step_layout(int D, int F, int TQ, int TV, int G, int N, int spw) {
  StepLayout L;
  auto tiles = [&](int T) { return (T + G - 1) / G; };
  int t = tiles(TQ);
  const int tpr = (3 * (kH / N) + 3) / 4;  // cluster variant: one rank's W_qkv tiles
  if (tpr > t) t = tpr;
  if (tiles(F / 2) > t) t = tiles(F / 2);
  if (tiles(D / 4) > t) t = tiles(D / 4);
  if (tiles(TV) > t) t = tiles(TV);
  L.max_rows = 4 * t;
  int part = kNumConsumerWarps * L.max_rows * 4;
  const int ws = kNumConsumerWarps * kPS * 4;  // attention warp states alias `part`
  if (ws > part) part = ws;
  if (3 * G * 4 > part) part = 3 * G * 4;  // flat O-phase merge: per-piece m, l, weight
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.xs = o;    o += r16((D > F ? D : F) * 2);
  L.part = o;  o += r16(part);
  L.gu = o;    o += r16(4 * tiles(F / 2) * 4);
  L.qf = o;    o += 3 * kH * 4 + kH * 2;  // q, k, v fp32 + fp16 A for the O projection
  L.dsm = o;   o += N * r16(3 * (kH / N) * 2) + N * r16((4 + kH) * 4);  // DSMEM gather | exchange
  L.red = o;   o += r16(kNumConsumerWarps * 4 * 2);
  L.tag = o;   o += r16(kNumSlots * 4);  // gate/up pool: tile index per ring slot (-1: end)
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

// Grid barrier with a precomputed target: the monotonic counter is k*G at
// launch (every earlier barrier completed), so target_n = base + n*G.  The
// arrival is a posted red.release (no atomic round trip on the critical
// path); thread 0 then polls with ld.acquire.
__device__ __forceinline__ void grid_sync(unsigned long long* counter, unsigned long long target,
                                          int tid) {
  // bar.sync orders every consumer's prior writes before thread 0's release
  // (cumulative), so one fence-carrying arrival per CTA publishes them all
  consumer_sync();
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(counter) : "memory");
    spin_until_geq(counter, target);
  }
  consumer_sync();
}

// thread 0 spins until *p >= target, then the CTA's consumers proceed
__device__ __forceinline__ void wait_counter(const unsigned long long* p, unsigned long long target,
                                             int tid) {
  if (tid == 0) {
    spin_until_geq(p, target);
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

// Work-stolen gate/up tail (the layered FFN kernel's CFB_DYN_POOL, here per
// layer inside the persistent step): after its static tiles each producer
// lane grabs whole tiles [T1s, T1s + pool) from a global counter and streams
// their pieces into its own consumer warp's sub-ring, tagging each slot with
// the tile; one failing grab per lane ends its pool (sentinel tag -1).  Each
// layer has its own counter and a launch adds exactly pool + 8 G to it, so
// floor(counter / per) * per read before this CTA's own failing grab is the
// launch's base: the value cannot reach the next multiple of per until every
// lane of every CTA (this one included) has failed.  (One shared counter is
// not enough: in a small model a producer can run a whole layer ahead of a
// CTA still waiting at a barrier.)
__device__ __forceinline__ void produce_pool(const Ring& ring, int lane, uint64_t pol, int& c,
                                            unsigned long long* ctr, int pool, int T1s,
                                            const char* w_gu, int tileB, int* tag) {
  const unsigned long long per = (unsigned long long)pool + 8ull * gridDim.x;
  const unsigned long long base = (ld_acquire_u64(ctr) / per) * per;
  const int npc = (tileB + kSlotBytes - 1) / kSlotBytes;
  bool done = lane >= kNumConsumerWarps;
  int cur = 0, piece = npc, nap = 32;
  while (true) {
    bool issued = false;
    if (!done) {
      const int sl = lane * ring.spw + (c % ring.spw);
      if (mbar_test(&ring.empty[sl], ((c / ring.spw) & 1) ^ 1)) {
        if (piece == npc) {
          const long long t = (long long)(atomicAdd(ctr, 1ull) - base);
          if (t >= pool) {
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
          bulk_g2s(ring.slot(sl), w_gu + (size_t)cur * tileB + b0, nb, &ring.full[sl], pol);
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

// Off-chip exchange (no-DSMEM ablation): every rank of the cluster stores its
// `bytes` from shared memory into its global slot (slot stride `stride`, byte
// offset `off`), the N ranks meet at a release/acquire counter, then each
// copies every peer's slot back into its own shared memory at dst(d, peer),
// d = the rotation distance (rank - peer) mod N, i.e. where the DSMEM push
// would have put it, so the math that follows is shared by both channels.
template <class Dst>
__device__ __forceinline__ void global_exchange(const void* src, int bytes, float* slots, int stride,
                                                int off, int rank, int N, unsigned long long* ctr,
                                                unsigned long long target, int tid, Dst&& dst) {
  char* mine = reinterpret_cast<char*>(slots) + (size_t)rank * stride + off;
  for (int v = tid; v < bytes / 16; v += kConsumerThreads)
    __stcg(reinterpret_cast<uint4*>(mine) + v, reinterpret_cast<const uint4*>(src)[v]);
  consumer_sync();  // thread 0's release below is cumulative over these stores
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_acquire_u64(ctr) < target) {
    }
  }
  consumer_sync();
  for (int d = 1; d < N; ++d) {
    const int peer = (rank - d + N) % N;
    const uint4* s = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(slots) +
                                                    (size_t)peer * stride + off);
    uint4* o = reinterpret_cast<uint4*>(dst(d, peer));
    for (int v = tid; v < bytes / 16; v += kConsumerThreads) o[v] = __ldcg(s + v);
  }
}

__device__ __forceinline__ void stamp(unsigned long long* tr, int k, int tid) {
  if (tr && tid == 0) tr[k] = globaltimer();
}

// kCluster = true: the attention module of head h runs on one thread-block
// cluster of N CTAs exactly as ClusterFusion's split_token dataflow (QKV
// slice GEMV -> DSMEM ClusterGather -> RoPE / KV append -> split-KV flash
// decoding -> one-round DSMEM (m, l, A) exchange -> O-projection slice), so
// the module has NO global dependency until the end-of-attention barrier.
// kCluster = false: flattened split over all SMs, partials exchanged through
// global memory with per-head counters (the ablation: same kernel, off-chip
// exchange instead of DSMEM).
//
// kDsmem = false (cluster variant only): the same cluster partitioning, but
// the ClusterGather and the (m, l, A) exchange go through global memory (a
// slot per rank, a per-cluster release/acquire counter) instead of DSMEM -
// the paper's "without DSMEM" ablation.
template <bool kCluster, bool kDsmem = true, bool kPaged = false>
__global__ void __launch_bounds__(kThreads, 1) llama_step_kernel(const StepParams p) {
  extern __shared__ __align__(128) char smem[];
  const int G = gridDim.x, i = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = p.D, F = p.F, nh = p.nh, N = p.N;
  const int hp = kH / N;                      // head dims per split_token rank
  const int TPH = N * p.tpr;                  // W_qkv tiles per head
  const int TQ = nh * TPH, T1 = F / 2, T2 = D / 4, TV = p.V / 4;
  const StepLayout Lo = step_layout(D, F, TQ, TV, G, N, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lo.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + Lo.misc + 16);  // [0] gather, [1] exchange

  const int S = *p.pos;
  // uniform across the grid: no barrier is entered.  Paged: the page that
  // receives row S must be reserved (rows < S were written by earlier steps)
  if (S + 1 > p.cap || (kPaged && __ldg(p.kv_pages + S / kPageRows) < 0)) {
    if (i == 0 && tid == 0) *p.err = 1;
    return;
  }
  const long long SP = S + 1;                 // attended positions per head
  // ---- static work assignment
  // cluster variant: cluster c = i / N serves heads c, c + C (rank r = i % N)
  const int C = G / N, cl = i / N, rank = i % N;
  const int nrounds = kCluster ? (cl < nh ? 1 + (cl + C < nh) : 0) : 0;
  const int seg = S == 0 ? 0 : (S + N - 1) / N;  // split_token KV segment (dataflows.py:109-114)
  const int s_lo = min(rank * seg, S), s_hi = min(s_lo + seg, S);
  const int cols = D / N;
  // flat variant ranges
  const long long PK = (long long)nh * SP;    // flattened (head, position) space
  const long long RO = (long long)nh * D;     // flattened (head, output column) rows
  const int q0 = kCluster ? 0 : (int)split_at(TQ, i, G), q1 = kCluster ? 0 : (int)split_at(TQ, i + 1, G);
  const long long k0 = split_at(PK, i, G), k1 = split_at(PK, i + 1, G);
  const long long o0 = split_at(RO, i, G), o1 = split_at(RO, i + 1, G);
  int ph[2] = {0, 0}, plo[2] = {0, 0}, phi[2] = {0, 0}, npiece = 0;
  int oh[2] = {0, 0}, olo[2] = {0, 0}, ohi[2] = {0, 0}, nopiece = 0;
  if (!kCluster) {
    for (long long x = k0; x < k1 && npiece < 2;) {  // attention pieces (head, [lo, hi))
      const int h = (int)(x / SP);
      const long long e = k1 < (h + 1) * SP ? k1 : (h + 1) * SP;
      ph[npiece] = h;
      plo[npiece] = (int)(x - h * SP);
      phi[npiece] = (int)(e - h * SP);
      ++npiece;
      x = e;
    }
    for (long long x = o0; x < o1 && nopiece < 2;) {  // O rows (head, [c_lo, c_hi))
      const int h = (int)(x / D);
      const long long e = o1 < (long long)(h + 1) * D ? o1 : (long long)(h + 1) * D;
      oh[nopiece] = h;
      olo[nopiece] = (int)(x - (long long)h * D);
      ohi[nopiece] = (int)(e - (long long)h * D);
      ++nopiece;
      x = e;
    }
  }
  // FFN and LM head: contiguous tile ranges over all G CTAs
  const int T1s = T1 - p.pool;  // gate/up tiles split statically; the rest is work-stolen
  const int a0 = (int)split_at(T1s, i, G), a1 = (int)split_at(T1s, i + 1, G);
  const int u0 = (int)split_at(T2, i, G), u1 = (int)split_at(T2, i + 1, G);
  const int v0 = (int)split_at(TV, i, G), v1 = (int)split_at(TV, i + 1, G);
  const int seg_bytes = r16(3 * hp * 2), pay_bytes = r16((4 + kH) * 4);

  if (tid == 0) {
    ring_init(ring);
    if (kCluster && N > 1) {
      mbar_init(&cbar[0], 1);
      mbar_arrive_expect_tx(&cbar[0], (N - 1) * seg_bytes);
      mbar_init(&cbar[1], 1);
      mbar_arrive_expect_tx(&cbar[1], (N - 1) * pay_bytes);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // no-DSMEM ablation: per-cluster exchange counter (monotonic; its launch
  // base is read before the start cluster barrier, i.e. before any increment)
  unsigned long long* xctr = p.counters + 2 * nh + cl;
  unsigned long long xtarget = (!kDsmem && kCluster) ? (ld_acquire_u64(xctr) / N) * N : 0ull;
  float* xslot = p.partials + (size_t)cl * N * ((seg_bytes + pay_bytes) / 4);  // [N][seg | pay]
  if (kCluster) cluster_arrive();  // peers' mbarriers initialised before any DSMEM push

  // The per-layer schedule, phase k of layer l computed on the fly (no arrays:
  // a dynamically indexed schedule would sit in local memory, which shares
  // the L1 with the 190+ KB ring).  Attention phases 0..5 (cluster: qkv, kv,
  // o per head round; flat: qkv, kv piece 0/1, o piece 0/1, -), FFN: 6
  // (gate/up), 7 (down).
  auto layer_phase = [&](int l, int k) -> Phase {
    if (k < 6) {
      if (kCluster) {
        const int j = k / 3, part_ = k % 3;
        const bool on = j < nrounds;
        const int h = cl + j * C;
        const size_t hr = on ? (size_t)h * N + rank : 0;
        if (part_ == 0)
          return make_phase(p.w_qkv[l] + hr * p.tpr * 4 * D, nullptr, on ? p.tpr : 0, 4 * D * 2, true);
        if (part_ == 1) {
          if (kPaged) {  // this head's rows of page 0 (layer_pphase adds the pages)
            const size_t hoff = on ? (size_t)h * p.kv_hstride : 0;
            return make_phase(p.k_cache[l] + hoff, p.v_cache[l] + hoff, on ? s_hi - s_lo : 0, kH * 2);
          }
          const size_t off = on ? ((size_t)h * p.cap + s_lo) * kH : 0;
          return make_phase(p.k_cache[l] + off, p.v_cache[l] + off, on ? s_hi - s_lo : 0, kH * 2);
        }
        return make_phase(p.w_out[l] + hr * cols * kH, nullptr, on ? cols : 0, kH * 2);
      }
      if (k == 0) return make_phase(p.w_qkv[l] + (size_t)q0 * 4 * D, nullptr, q1 - q0, 4 * D * 2, true);
      if (k <= 2) {
        const int j = k - 1;
        const int n = j < npiece ? (phi[j] < S ? phi[j] : S) - plo[j] : 0;
        const size_t off = ((size_t)ph[j] * p.cap + (j < npiece ? plo[j] : 0)) * kH;
        return make_phase(p.k_cache[l] + off, p.v_cache[l] + off, n > 0 ? n : 0, kH * 2);
      }
      if (k <= 4) {
        // W_out [head][rank][cols][H] flattens to [head][column][H]
        const int j = k - 3;
        const size_t off = ((size_t)oh[j] * D + (j < nopiece ? olo[j] : 0)) * kH;
        return make_phase(p.w_out[l] + off, nullptr, j < nopiece ? ohi[j] - olo[j] : 0, kH * 2);
      }
      return make_phase(nullptr, nullptr, 0, 16);
    }
    if (k == 6) return make_phase(p.w_gu[l] + (size_t)a0 * 4 * D, nullptr, a1 - a0, 4 * D * 2, true);
    return make_phase(p.w_dn[l] + (size_t)u0 * 4 * F, nullptr, u1 - u0, 4 * F * 2, true);
  };
  // the producer's view: the KV phases (cluster variant, k % 3 == 1) read the
  // page pool through the block table when the cache is paged
  auto layer_pphase = [&](int l, int k) -> PagedPhase {
    const Phase ph_ = layer_phase(l, k);
    if (kPaged && k < 6 && k % 3 == 1)
      return paged_phase(ph_, p.kv_pages, s_lo, p.kv_pstride * 2);
    return paged_phase(ph_);
  };
  // At a barrier the ring (ring_bytes) already holds the head of the next
  // phase and stalls once full; thread 0 lets HBM keep working on the bytes
  // after it by prefetching the next `l2_prefetch` bytes of that phase into
  // L2 (the producer's bulk copies then hit L2).  Rows/tiles are contiguous
  // from src0, so the ring holds exactly the first ring_bytes of the phase.
  auto prefetch_next = [&](const Phase& P) {
    if (tid != 0 || p.l2_prefetch <= 0 || P.src1) return;
    const long long total = (long long)P.n_units * P.unit_bytes;
    const long long lo = ring_bytes(p.spw), hi = min(total, lo + (long long)p.l2_prefetch);
    for (long long o = lo; o < hi; o += 16384)
      bulk_prefetch_l2(P.src0 + o, (uint32_t)min(16384ll, hi - o) & ~15u);
  };

  if (warp == kNumConsumerWarps) {  // ---------------------------- producer
    const uint64_t pol = policy_evict_first();
    int c = 0;
    int* tag = reinterpret_cast<int*>(smem + Lo.tag);
    // paged KV: the block-table entries of this CTA's segment pages, in the
    // producer lanes' registers for the whole launch (produce_gen_paged)
    int pgr[kPageRegs];
    const int p0 = s_lo / kPageRows;
#pragma unroll
    for (int k = 0; k < kPageRegs; ++k)
      pgr[k] = kPaged && (p0 + 32 * k + lane) * kPageRows < p.cap ? __ldg(p.kv_pages + p0 + 32 * k + lane) : 0;
    for (int l = 0; l < p.L; ++l) {
      if constexpr (kPaged)
        produce_gen_paged(7, [&](int k) { return layer_pphase(l, k); }, ring, lane, pol, c, pgr, p0);
      else
        produce_gen(7, [&](int k) { return layer_phase(l, k); }, ring, lane, pol, c);
      if (p.pool > 0)
        produce_pool(ring, lane, pol, c, p.pool_ctr + l, p.pool, T1s,
                     reinterpret_cast<const char*>(p.w_gu[l]), 4 * D * 2, tag);
      produce_gen(1, [&](int) { return layer_phase(l, 7); }, ring, lane, pol, c);
    }
    produce_gen(1, [&](int) { return make_phase(p.lm_head + (size_t)v0 * 4 * D, nullptr, v1 - v0, 4 * D * 2, true); },
                ring, lane, pol, c);
    __syncwarp();
    if (kCluster) {  // both cluster-barrier phases of the CTA (start, end)
      cluster_wait();
      cluster_arrive();
      cluster_wait();
    }
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
  __half* gseg = reinterpret_cast<__half*>(smem + Lo.dsm);                 // [N][seg]
  float* pay = reinterpret_cast<float*>(smem + Lo.dsm + N * seg_bytes);    // [N][4 + H]
  float* red = reinterpret_cast<float*>(smem + Lo.red);
  unsigned* last = reinterpret_cast<unsigned*>(smem + Lo.misc);
  unsigned long long* qkv_done = p.counters;
  unsigned long long* att_done = p.counters + nh;

  // embed: resid[c] = embed[token][c] for this CTA's slice; counters reset
  const bool tp = p.T > 1;
  const int c0 = (int)split_at(D, i, G), c1 = (int)split_at(D, i + 1, G);  // this CTA's D slice
  // this rank's sums: its NVLS copy, or its own exchange block
  unsigned long long* xown = tp ? (p.uc_sum ? p.uc_sum : p.xch[p.trank]) : nullptr;
  {
    const int tok = *p.token;
    for (int c = c0 + tid; c < c1; c += kConsumerThreads) {
      p.resid[c] = __half2float(p.embed[(size_t)tok * D + c]);
      if (tp) {  // set 0 (layer 0's sums) starts at zero; set 1 is zeroed by layer 0
        tp_xa(xown, D, 0)[c] = 0ull;
        tp_xf(xown, D, 0)[c] = 0ull;
      }
    }
    if (!kCluster && i == 0 && tid < 2 * nh) p.counters[tid] = 0ull;
    if (tp && i == 0 && tid == 0) *tp_key(xown, D) = 0ull;
  }
  // barrier bases: no CTA can pass the first barrier before all have read them
  // (cross-rank: the count is below base + T G until this CTA arrives)
  unsigned long long bar_target = (ld_acquire_u64(p.barrier) / G) * G;
  const unsigned long long TG = (unsigned long long)p.T * G;
  unsigned long long x_target = tp ? (ld_acquire_sys_u64(tp_bar(xown, D)) / TG) * TG : 0ull;
  const unsigned long long tok_base =
      tp ? (ld_acquire_sys_u64(tp_tok(xown, D)) / p.T) * p.T : 0ull;
  if (kCluster) cluster_wait();
  if (tp) {
    cross_sync(p, x_target += TG, tid);  // no rank pushes into set 0 before it is zeroed everywhere
  } else {
    bar_target += G;
    grid_sync(p.barrier, bar_target, tid);
  }

  // cross-CTA data is read through L2 (ld.global.cg): L1 is not coherent
  const float* resid_g = p.resid;
  // residual stream h_l entering layer l (l == L: the final norm's input).
  // Single GPU: resid, updated in place by the down-projection epilogue.
  // TP: H[(l-1) & 1] + XA[(l-1) % 3] + XF[(l-1) % 3] (H[0] = embed for l == 0).
  auto h_in = [&](int l, int v) -> float4 {
    if (!tp || l == 0) return __ldcg(reinterpret_cast<const float4*>(resid_g) + v);
    const float* Hp = ((l - 1) & 1) ? p.resid2 : p.resid;
    const float4 r = __ldcg(reinterpret_cast<const float4*>(Hp) + v);
    const ulonglong2* xa = reinterpret_cast<const ulonglong2*>(tp_xa(xown, D, (l - 1) % 3));
    const ulonglong2* xf = reinterpret_cast<const ulonglong2*>(tp_xf(xown, D, (l - 1) % 3));
    const ulonglong2 a0 = __ldcg(xa + 2 * v), a1 = __ldcg(xa + 2 * v + 1);
    const ulonglong2 f0 = __ldcg(xf + 2 * v), f1 = __ldcg(xf + 2 * v + 1);
    return make_float4(__fadd_rn(__fadd_rn(r.x, fixed_to_float(a0.x)), fixed_to_float(f0.x)),
                       __fadd_rn(__fadd_rn(r.y, fixed_to_float(a0.y)), fixed_to_float(f0.y)),
                       __fadd_rn(__fadd_rn(r.z, fixed_to_float(a1.x)), fixed_to_float(f1.x)),
                       __fadd_rn(__fadd_rn(r.w, fixed_to_float(a1.y)), fixed_to_float(f1.y)));
  };
  // TP, layer l >= 1: the slice owner stores h_l into H[l & 1] (read by this
  // layer's FFN prologue) and zeroes its slice of set (l + 1) % 3
  auto tp_layer_start = [&](int l) {
    if (!tp) return;
    float* Hn = (l & 1) ? p.resid2 : p.resid;
    const float* Hp = ((l - 1) & 1) ? p.resid2 : p.resid;
    for (int c = c0 + tid; c < c1; c += kConsumerThreads) {
      if (l > 0)
        Hn[c] = __fadd_rn(__fadd_rn(__ldcg(Hp + c), fixed_to_float(__ldcg(tp_xa(xown, D, (l - 1) % 3) + c))),
                          fixed_to_float(__ldcg(tp_xf(xown, D, (l - 1) % 3) + c)));
      tp_xa(xown, D, (l + 1) % 3)[c] = 0ull;
      tp_xf(xown, D, (l + 1) % 3)[c] = 0ull;
    }
  };
  unsigned long long* accA = p.accA;
  int cnt = 0;
  int use = 0;  // DSMEM barrier phase (one gather + one exchange per head round)
  const int g = lane / kLPK, li = lane % kLPK;
  const float scale = p.inv_sqrt_h;
  const int half = kH / 2;

  // RoPE of q and k_new at position S (rotate-half), fp16-stored values
  // the position is fixed for the whole launch: thread d < H/2 keeps its
  // rotation (cos, sin) in registers instead of re-reading the table in
  // every layer's attention critical path
  const float rope_c = tid < half ? p.rope_cs[((size_t)S * half + tid) * 2] : 0.f;
  const float rope_s = tid < half ? p.rope_cs[((size_t)S * half + tid) * 2 + 1] : 0.f;
  auto rope_qk = [&]() {
    for (int d = tid; d < half; d += kConsumerThreads) {  // half <= kConsumerThreads: d == tid
      const float c = rope_c, sn = rope_s;
      const float q1_ = qf[d], q2 = qf[d + half], k1_ = kf[d], k2 = kf[d + half];
      qf[d] = round_to<__half>(__fsub_rn(__fmul_rn(q1_, c), __fmul_rn(q2, sn)));
      qf[d + half] = round_to<__half>(__fadd_rn(__fmul_rn(q2, c), __fmul_rn(q1_, sn)));
      kf[d] = round_to<__half>(__fsub_rn(__fmul_rn(k1_, c), __fmul_rn(k2, sn)));
      kf[d + half] = round_to<__half>(__fadd_rn(__fmul_rn(k2, c), __fmul_rn(k1_, sn)));
    }
    consumer_sync();
  };
  auto append_kv = [&](int l, int h) {  // KV-cache append at row S (read by later steps only)
    const size_t off = kPaged
        ? (size_t)h * p.kv_hstride + (size_t)__ldg(p.kv_pages + S / kPageRows) * p.kv_pstride +
              (size_t)(S % kPageRows) * kH
        : ((size_t)h * p.cap + S) * kH;
    for (int d = tid; d < kH; d += kConsumerThreads) {
      p.k_cache[l][off + d] = __float2half_rn(kf[d]);
      p.v_cache[l][off + d] = __float2half_rn(vf[d]);
    }
  };
  // flash decoding of this CTA's KV rows (+ the new token when has_new) and
  // the in-order merge of the 8 warp states -> (m, l, A) in `out` (fp32)
  auto attend_rows = [&](const Phase& PKV, bool has_new, float* out) {
    float q[kEPL], acc[kEPL], m = -INFINITY, lsum = 0.f;
#pragma unroll
    for (int e = 0; e < kEPL; ++e) {
      q[e] = qf[li * kEPL + e];
      acc[e] = 0.f;
    }
    consume_phase(PKV, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
      const __half* K = reinterpret_cast<const __half*>(slot);
      const __half* V = reinterpret_cast<const __half*>(slot + kSlotBytes / 2);
      attend(q, m, lsum, acc, it.nunits, g, scale,
             [&](int k, float* o) { load_elems<__half, kEPL>(K + k * kH + li * kEPL, o); },
             [&](int k, float* o) { load_elems<__half, kEPL>(V + k * kH + li * kEPL, o); });
    });
    if (has_new && warp == 0)  // the new token's K/V: attended exactly once
      attend(q, m, lsum, acc, 1, g, scale,
             [&](int, float* o) {
#pragma unroll
               for (int e = 0; e < kEPL; ++e) o[e] = kf[li * kEPL + e];
             },
             [&](int, float* o) {
#pragma unroll
               for (int e = 0; e < kEPL; ++e) o[e] = vf[li * kEPL + e];
             });
#pragma unroll
    for (int o = kLPK; o < 32; o <<= 1) {  // fold the key groups (same dims, shared m)
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
      out[4 + d] = a;
      if (d == 0) {
        out[0] = mm;
        out[1] = ll;
      }
    }
  };

  for (int l = 0; l < p.L; ++l) {
    unsigned long long* tr = p.trace ? p.trace + ((size_t)l * G + i) * 8 : nullptr;
    stamp(tr, 0, tid);
    if (kCluster) {
      // ================= attention module on the cluster (split_token, Alg. 3)
      tp_layer_start(l);
      if (nrounds > 0)
        rmsnorm_to_smem_ld<__half, true>(xs, [&](int, int v) { return h_in(l, v); }, p.attn_norm[l], 1, D,
                                         p.eps, red, tid);
      for (int j = 0; j < nrounds; ++j, ++use) {
        const int h = cl + j * C;
        // 1. QKV GEMV of this rank's q|k|v slices (dataflows.py:256-267)
        tiled_gemv_phase<__half, 1, true>(layer_phase(l, 3 * j), ring, warp, lane, tid, cnt, xs, D, 1, 4 * p.tpr,
                                          part, [&](int row, int, float v) {
                                            if (row < 3 * hp) gseg[row] = __float2half_rn(v);
                                          });
        consumer_sync();
        stamp(tr, 1, tid);
        // 2. ClusterGather (one round, rank-rotated slots, dataflows.py:268-279)
        if (kDsmem && warp == 0 && N > 1) {
          for (int d = 1; d < N; ++d)
            dsmem_push(gseg, reinterpret_cast<char*>(gseg) + d * seg_bytes, &cbar[0], seg_bytes,
                       (rank + d) % N, lane);
          __syncwarp();
          mbar_wait(&cbar[0], use & 1);
          if (lane == 0) mbar_arrive_expect_tx(&cbar[0], (N - 1) * seg_bytes);  // next round
        }
        if (!kDsmem && N > 1) {  // off-chip: slot store, counter meet, peers' slots back via L2
          global_exchange(gseg, seg_bytes, xslot, seg_bytes + pay_bytes, 0, rank, N, xctr,
                          xtarget += N, tid,
                          [&](int d, int) { return reinterpret_cast<char*>(gseg) + d * seg_bytes; });
        }
        consumer_sync();
        for (int d = tid; d < kH; d += kConsumerThreads) {
          const int rr = d / hp, ii = d % hp;
          const __half* sg = gseg + ((rank - rr + N) % N) * (seg_bytes / 2);
          qf[d] = __half2float(sg[ii]);
          kf[d] = __half2float(sg[hp + ii]);
          vf[d] = __half2float(sg[2 * hp + ii]);
        }
        consumer_sync();
        // 3. RoPE + KV append (rank N-1 owns the new row)
        rope_qk();
        if (rank == N - 1) append_kv(l, h);
        // 4. flash decoding over this rank's segment; new token on rank N-1
        float* mine = pay + rank * (pay_bytes / 4);
        attend_rows(layer_phase(l, 3 * j + 1), rank == N - 1, mine);
        consumer_sync();
        stamp(tr, 2, tid);
        // 5. one-round DSMEM exchange of fp32 (m, l, A), merged in rank order
        //    (= MAX-reduce, rescale, SUM-reduce, rescale, SUM-reduce; dataflows.py:187-232)
        if (kDsmem && warp == 0 && N > 1) {
          for (int d = 1; d < N; ++d) dsmem_push(mine, mine, &cbar[1], pay_bytes, (rank + d) % N, lane);
          __syncwarp();
          mbar_wait(&cbar[1], use & 1);
          if (lane == 0) mbar_arrive_expect_tx(&cbar[1], (N - 1) * pay_bytes);
        }
        if (!kDsmem && N > 1) {
          global_exchange(mine, pay_bytes, xslot, seg_bytes + pay_bytes, seg_bytes, rank, N, xctr,
                          xtarget += N, tid, [&](int, int r2) {
                            return reinterpret_cast<char*>(pay + r2 * (pay_bytes / 4));
                          });
        }
        consumer_sync();
        for (int d = tid; d < kH; d += kConsumerThreads) {
          float ms = -INFINITY;
          for (int r2 = 0; r2 < N; ++r2) ms = fmaxf(ms, pay[r2 * (pay_bytes / 4)]);
          float ls = 0.f, a = 0.f;
          for (int r2 = 0; r2 < N; ++r2) {
            const float* src = pay + r2 * (pay_bytes / 4);
            const float f = (src[0] == -INFINITY) ? 0.f : expf(src[0] - ms);
            ls = fmaf(src[1], f, ls);
            a = fmaf(src[4 + d], f, a);
          }
          abuf[d] = __float2half_rn(__fdiv_rn(a, ls));
        }
        consumer_sync();
        // 6. O-projection of this rank's D/N output columns -> fixed-point head sum
        consume_phase(layer_phase(l, 3 * j + 2), ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
          rowlane_item<__half, 1>(it, slot, abuf, kH, 1, lane, [&](int gcol, const float (&s)[1]) {
            red_add_fixed(&accA[rank * cols + gcol], s[0]);
          });
        });
      }
      if (nrounds == 0) {
        stamp(tr, 1, tid);
        stamp(tr, 2, tid);
      }
      stamp(tr, 3, tid);
    } else {
      // ================= flattened attention over all SMs, global exchange
      tp_layer_start(l);
      rmsnorm_to_smem_ld<__half, true>(xs, [&](int, int v) { return h_in(l, v); }, p.attn_norm[l], 1, D,
                                       p.eps, red, tid);
      tiled_gemv_phase<__half, 1, true>(layer_phase(l, 0), ring, warp, lane, tid, cnt, xs, D, 1, 4 * (q1 - q0), part,
                                        [&](int row, int, float v) {
                                          p.qkv[(size_t)4 * q0 + row] = __float2half_rn(v);
                                        });
      consumer_sync();  // thread 0's releases are cumulative over the CTA's q|k|v stores
      if (tid == 0) {
        for (int h = q0 / TPH; h < nh && h * TPH < q1; ++h) {
          const int lo = max(q0, h * TPH), hi = min(q1, (h + 1) * TPH);
          red_release_add(&qkv_done[h], (unsigned long long)(hi - lo));
        }
      }
      stamp(tr, 1, tid);
      for (int j = 0; j < npiece; ++j) {
        const int h = ph[j];
        const bool has_new = phi[j] == S + 1;
        wait_counter(&qkv_done[h], (unsigned long long)TPH * (l + 1), tid);
        for (int d = tid; d < kH; d += kConsumerThreads) {  // q, k_new, v_new of head h
          const size_t r = ((size_t)h * N + d / hp) * p.tpr * 4 + d % hp;
          qf[d] = __half2float(__ldcg(p.qkv + r));
          kf[d] = __half2float(__ldcg(p.qkv + r + hp));
          vf[d] = __half2float(__ldcg(p.qkv + r + 2 * hp));
        }
        consumer_sync();
        rope_qk();
        if (has_new) append_kv(l, h);
        attend_rows(layer_phase(l, 1 + j), has_new, p.partials + ((size_t)h * G + i) * kPS);
        consumer_sync();
        if (tid == 0) red_release_add(&att_done[h], 1ull);
      }
      stamp(tr, 2, tid);
      for (int j = 0; j < nopiece; ++j) {  // merge + O projection
        const int h = oh[j];
        const long long ha = (long long)h * SP, hb = ha + SP;
        const int first = owner_of(ha, PK, G), lastc = owner_of(hb - 1, PK, G);
        const int ncand = lastc - first + 1;  // CTAs whose (head, position) range may touch head h
        // per-piece (m, l) into smem in parallel (a piece = a CTA with a non-empty range),
        // then every thread merges its dims over the pieces in ascending CTA order
        float* pm = part;          // [ncand] m
        float* pl = part + G;      // [ncand] l
        float* pw = part + 2 * G;  // [ncand] weights e^(m_c - M) (0: empty / -inf piece)
        int npieces = 0;
        for (int c = first; c <= lastc; ++c) npieces += split_at(PK, c, G) < split_at(PK, c + 1, G);
        wait_counter(&att_done[h], (unsigned long long)npieces * (l + 1), tid);
        for (int t = tid; t < ncand; t += kConsumerThreads) {
          const int c = first + t;
          const bool ne = split_at(PK, c, G) < split_at(PK, c + 1, G);
          const float* src = p.partials + ((size_t)h * G + c) * kPS;
          pm[t] = ne ? __ldcg(src) : -INFINITY;
          pl[t] = ne ? __ldcg(src + 1) : 0.f;
        }
        consumer_sync();
        {
          float ms = -INFINITY;
          for (int t = 0; t < ncand; ++t) ms = fmaxf(ms, pm[t]);
          for (int t = tid; t < ncand; t += kConsumerThreads) pw[t] = pm[t] == -INFINITY ? 0.f : expf(pm[t] - ms);
        }
        consumer_sync();
        for (int d = tid; d < kH; d += kConsumerThreads) {
          float ls = 0.f, a = 0.f;
          for (int t0 = 0; t0 < ncand; t0 += 8) {  // 8 independent L2 loads in flight
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              v[k] = (t0 + k < ncand && pw[t0 + k] != 0.f)
                         ? __ldcg(p.partials + ((size_t)h * G + first + t0 + k) * kPS + 4 + d)
                         : 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (t0 + k < ncand && pw[t0 + k] != 0.f) {  // fixed (ascending) order: deterministic
                ls = fmaf(pl[t0 + k], pw[t0 + k], ls);
                a = fmaf(v[k], pw[t0 + k], a);
              }
          }
          abuf[d] = __float2half_rn(__fdiv_rn(a, ls));
        }
        consumer_sync();
        const int c_lo = olo[j];
        consume_phase(layer_phase(l, 3 + j), ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
          // absolute column: packed rows are chunk-rotated by their row within the
          // rank slice, (c mod D/N) mod 16 == c mod 16 (host-checked)
          Item it2 = it;
          it2.unit0 += c_lo;
          rowlane_item<__half, 1>(it2, slot, abuf, kH, 1, lane, [&](int col, const float (&s)[1]) {
            red_add_fixed(&accA[col], s[0]);
          });
        });
      }
      stamp(tr, 3, tid);
    }
    prefetch_next(layer_phase(l, 6));
    bar_target += G;
    grid_sync(p.barrier, bar_target, tid);
    if (tp) {  // attention all-reduce: this CTA's slice of the local head sum to every rank
      for (int c = c0 + tid; c < c1; c += kConsumerThreads) {
        const unsigned long long v = __ldcg(accA + c);
        tp_push(p, l % 3, c, v);  // tp_xa set l % 3
        accA[c] = 0ull;
      }
      cross_sync(p, x_target += TG, tid);
    }
    stamp(tr, 4, tid);

    // ---- FFN gate/up with the residual + head-sum RMSNorm prologue
    rmsnorm_to_smem_ld<__half, true>(
        xs,
        [&](int, int v) {
          const float* Hl = tp && (l & 1) ? p.resid2 : resid_g;  // TP: h_l in H[l & 1]
          const ulonglong2* acc = reinterpret_cast<const ulonglong2*>(tp ? tp_xa(xown, D, l % 3) : accA);
          const float4 r = __ldcg(reinterpret_cast<const float4*>(Hl) + v);
          const ulonglong2 x0 = __ldcg(acc + 2 * v);
          const ulonglong2 x1 = __ldcg(acc + 2 * v + 1);
          return make_float4(__fadd_rn(r.x, fixed_to_float(x0.x)), __fadd_rn(r.y, fixed_to_float(x0.y)),
                             __fadd_rn(r.z, fixed_to_float(x1.x)), __fadd_rn(r.w, fixed_to_float(x1.y)));
        },
        p.ffn_norm[l], 1, D, p.eps, red, tid);
    tiled_gemv_phase<__half, 1, true>(layer_phase(l, 6), ring, warp, lane, tid, cnt, xs, D, 1,
                                      4 * (a1 - a0), part, [&](int row, int, float v) { gu[row] = v; });
    consumer_sync();
    for (int jj = tid; jj < 2 * (a1 - a0); jj += kConsumerThreads) {
      const int t = jj >> 1, e = jj & 1;  // tile rows: g0 g1 u0 u1
      const float gt = gu[4 * t + e], up = gu[4 * t + 2 + e];
      const float sl = __fdiv_rn(gt, __fadd_rn(1.0f, expf(-gt)));
      p.act[2 * a0 + jj] = __float2half_rn(__fmul_rn(sl, up));
    }
    if (p.pool > 0) {
      // work-stolen tiles: whole tiles (npc pieces in this warp's consecutive
      // slots); lanes 0..3 accumulate rows (gate 2t, gate 2t+1, up 2t, up 2t+1)
      const int* tag = reinterpret_cast<const int*>(smem + Lo.tag);
      const int tileB = 4 * D * 2, npc = (tileB + kSlotBytes - 1) / kSlotBytes;
      const Phase P6 = layer_phase(l, 6);
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
          tile_item<__half, 1, true>(P6, it, ring.slot(s2), xs, D, 1, lane,
                                     [&](int, const float (&sm)[1]) { rowsum += sm[0]; });
          __syncwarp();
          if (lane == 0) mbar_arrive(&ring.empty[s2]);
          ++cnt;
        }
        const float up = __shfl_sync(0xffffffffu, rowsum, (lane & 1) + 2);
        if (lane < 2) {
          const float sl2 = __fdiv_rn(rowsum, __fadd_rn(1.0f, expf(-rowsum)));
          p.act[2 * t + lane] = __float2half_rn(__fmul_rn(sl2, up));
        }
      }
    }
    stamp(tr, 5, tid);
    prefetch_next(layer_phase(l, 7));
    bar_target += G;
    grid_sync(p.barrier, bar_target, tid);

    // ---- down projection + residual: resid = resid + head sum + FFN
    load_act_to_smem<__half, true>(xs, p.act, 1, F, tid);
    stamp(tr, 6, tid);
    tiled_gemv_phase<__half, 1, true>(layer_phase(l, 7), ring, warp, lane, tid, cnt, xs, F, 1,
                                      4 * (u1 - u0), part, [&](int row, int, float v) {
                                        const int c = 4 * u0 + row;
                                        if (tp) {  // FFN all-reduce: partial column sums to every rank
                                          const unsigned long long q =
                                              (unsigned long long)__float2ll_rn(v * 4294967296.0f);
                                          tp_push(p, 3 + l % 3, c, q);  // tp_xf set l % 3
                                          return;
                                        }
                                        const float r = __fadd_rn(__ldcg(p.resid + c),
                                                                  fixed_to_float(__ldcg(accA + c)));
                                        accA[c] = 0ull;
                                        p.resid[c] = __fadd_rn(r, v);
                                      });
    if (l + 1 < p.L)
      prefetch_next(layer_phase(l + 1, 0));
    else
      prefetch_next(make_phase(p.lm_head + (size_t)v0 * 4 * D, nullptr, v1 - v0, 4 * D * 2, true));
    if (tp) {
      cross_sync(p, x_target += TG, tid);
    } else {
      bar_target += G;
      grid_sync(p.barrier, bar_target, tid);
    }
    stamp(tr, 7, tid);
  }

  // ---- final RMSNorm + LM head + argmax
  rmsnorm_to_smem_ld<__half, true>(xs, [&](int, int v) { return h_in(p.L, v); }, p.final_norm, 1, D, p.eps,
                                   red, tid);
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
  if (*last) {
    // the G per-CTA candidates, reduced in parallel: thread c loads
    // candidate c (one round trip), warp shuffles, then warp 0 folds the
    // warp winners; `better` is a total order (value, then lower index), so
    // the winner does not depend on the reduction tree
    if (tid == 0) __threadfence();
    consumer_sync();
    float v = -INFINITY;
    int ix = 0x7fffffff;
    for (int c = tid; c < G; c += kConsumerThreads) {
      const float cv = __ldcg(&p.cand_val[c]);
      const int ci = __ldcg(&p.cand_idx[c]);
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
    if (lane == 0) {
      red[warp] = v;
      reinterpret_cast<int*>(red)[kNumConsumerWarps + warp] = ix;
    }
    consumer_sync();
    if (tid == 0) {  // fold the warp winners, publish the token
      v = -INFINITY;
      ix = 0x7fffffff;
      for (int w2 = 0; w2 < kNumConsumerWarps; ++w2)
        if (better(red[w2], reinterpret_cast<int*>(red)[kNumConsumerWarps + w2], v, ix)) {
          v = red[w2];
          ix = reinterpret_cast<int*>(red)[kNumConsumerWarps + w2];
        }
      if (tp) {  // global argmax over the vocabulary shards: MAX of order-preserving keys
        const unsigned long long key = argmax_key(v, ix + p.voff);
        for (int t = 0; t < p.T; ++t) red_max_u64(tp_key(p.xch[t], D), key);
        __threadfence_system();
        for (int t = 0; t < p.T; ++t) red_release_sys_add(tp_tok(p.xch[t], D), 1ull);
        tp_spin(tp_tok(xown, D), tok_base + p.T, p.timeout_ns, p.err);
        const unsigned long long k = ld_acquire_sys_u64(tp_key(xown, D));
        ix = (int)(0xFFFFFFFFu - (unsigned)(k & 0xFFFFFFFFull));
      }
      *p.token = ix;
      *p.ticket = 0;
      *p.pos = S + 1;
    }
  }
  if (kCluster) {
    cluster_arrive();  // no CTA leaves while a peer could still address its smem
    cluster_wait();
  }
}

}  // namespace

size_t tp_xch_bytes(int hidden) { return (6 * (size_t)hidden + 48) * 8; }

int llama_step_smem(int D, int F, int nh, int N, int tpr, int V, int G, int max_spw, int* spw_out) {
  int spw = tuned_spw();
  if (max_spw > 0 && max_spw < spw) spw = max_spw;
  const int TQ = nh * N * tpr, TV = V / 4;
  StepLayout L = step_layout(D, F, TQ, TV, G, N, spw);
  while (L.total > kMaxSmem && spw > 1) L = step_layout(D, F, TQ, TV, G, N, --spw);
  if (spw_out) *spw_out = spw;
  return L.total;
}

static int step_check(const LlamaStepArgs* a) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->head_dim != kH) return set_error(CFB_ERR_DIMENSION, "persistent engine needs head_dim 128");
  const int N = a->cluster;
  if (N < 1 || N > 16 || (N & (N - 1)) || kH % N)
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16]");
  if (a->hidden % 8 || a->inter % 8 || a->vocab % 4 || (a->hidden / N) % (kH * 2 / 16))
    return set_error(CFB_ERR_DIMENSION, "persistent engine: hidden/inter multiples of 8, vocab of 4");
  return CFB_OK;
}

// Grid of the persistent launch: every CTA must be co-resident (grid
// barriers).  Flat: one CTA per SM.  Cluster: as many N-CTA clusters as the
// GPCs can hold at once (cudaOccupancyMaxActiveClusters; 33 x 4 = 132 SMs on a
// B200 at ~225 KB of shared memory per CTA).
int llama_step_grid(const LlamaStepArgs* a, int* grid_out, int* smem_out, int* spw_out) {
  if (const int rc = step_check(a)) return rc;
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int N = a->cluster, tpr = (3 * (kH / N) + 3) / 4;
  int G = a->grid > 0 && a->grid < sms ? a->grid : sms;
  int spw = 0;
  int smem = llama_step_smem(a->hidden, a->inter, a->n_heads, N, tpr, a->vocab, G, a->ring_spw, &spw);
  if (a->cluster_attn) {
    const void* kern = (const void*)llama_step_kernel<true>;
    if (const int rc = configure_kernel(kern, kMaxSmem, true)) return rc;
    for (int it = 0; it < 3; ++it) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G - G % N, 1, 1);
      cfg.blockDim = dim3(kThreads, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = N;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      CFB_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
      const int G2 = nc * N < G ? nc * N : G - G % N;
      if (G2 < N) return set_error(CFB_ERR_SMEM, "persistent engine: no cluster of %d fits", N);
      if (G2 == G) break;
      G = G2;
      smem = llama_step_smem(a->hidden, a->inter, a->n_heads, N, tpr, a->vocab, G, a->ring_spw, &spw);
    }
  }
  if (!a->cluster_attn && G < a->n_heads)  // flattened ranges then span at most two heads
    return set_error(CFB_ERR_DIMENSION, "persistent engine: grid %d vs %d heads", G, a->n_heads);
  if (a->cluster_attn && 2 * (G / N) < a->n_heads)
    return set_error(CFB_ERR_DIMENSION, "persistent engine: %d clusters for %d heads", G / N, a->n_heads);
  if (smem > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "persistent engine needs %d B of shared memory (max %d)", smem,
                     kMaxSmem);
  if (grid_out) *grid_out = G;
  if (smem_out) *smem_out = smem;
  if (spw_out) *spw_out = spw;
  return CFB_OK;
}

int llama_step_launch(const LlamaStepArgs* a, cudaStream_t st) {
  int G = 0, smem = 0, spw = 0;
  if (const int rc = llama_step_grid(a, &G, &smem, &spw)) return rc;
  const int N = a->cluster;
  StepParams p;
  p.L = a->n_layers;
  p.D = a->hidden;
  p.nh = a->n_heads;
  p.F = a->inter;
  p.V = a->vocab;
  p.cap = a->cache_cap;
  p.N = N;
  p.tpr = (3 * (kH / N) + 3) / 4;
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
  p.kv_pages = a->kv_pages;
  p.kv_pstride = a->kv_pstride;
  p.kv_hstride = a->kv_hstride;
  if (p.kv_pages && !a->cluster_attn)
    return set_error(CFB_ERR_ARGUMENT, "paged KV needs the cluster attention (persistent / nodsmem engine)");
  // a CTA's segment (ceil(cap / N) rows, any offset) must fit the producer's page registers
  if (p.kv_pages && ((a->cache_cap + N - 1) / N + kPageRows - 1) / kPageRows + 1 >= 32 * kPageRegs)
    return set_error(CFB_ERR_DIMENSION, "paged KV: %d positions over clusters of %d exceed %d pages per CTA",
                     a->cache_cap, N, 32 * kPageRegs - 2);
  p.embed = static_cast<const __half*>(a->embed);
  p.final_norm = static_cast<const __half*>(a->final_norm);
  p.lm_head = static_cast<const __half*>(a->lm_head);
  p.rope_cs = a->rope_cs;
  p.resid = a->resid;
  p.accA = a->accA;
  p.act = static_cast<__half*>(a->act);
  p.qkv = static_cast<__half*>(a->qkv);
  p.partials = a->partials;
  p.barrier = a->barrier;
  p.counters = a->counters;
  p.pool_ctr = a->pool_ctr;
  const int ppc = a->pool_per_cta > 0 ? a->pool_per_cta : 4;
  p.pool = a->pool_ctr ? (ppc * G < a->inter / 8 ? ppc * G : a->inter / 8) : 0;
  p.logits = a->logits;
  p.cand_val = a->cand_val;
  p.cand_idx = a->cand_idx;
  p.ticket = a->ticket;
  p.token = a->token;
  p.pos = a->pos;
  p.err = a->err;
  p.trace = a->trace;
  p.T = a->tp_size > 1 ? a->tp_size : 1;
  p.trank = a->tp_rank;
  p.voff = a->vocab_offset;
  p.xch = a->xch;
  p.resid2 = a->resid2;
  p.uc_sum = a->uc_sum;
  p.mc_sum = a->mc_sum;
  p.timeout_ns = a->timeout_ns;
  p.l2_prefetch = a->l2_prefetch;
  if (p.T > 1 && (!p.xch || !p.resid2 || p.trank < 0 || p.trank >= p.T))
    return set_error(CFB_ERR_ARGUMENT, "tensor-parallel step without exchange blocks");
  // emulated ranks share the GPU: every rank's grid is resident by construction
  // (the caller sizes it), a cooperative launch could not overlap with the peers'
  const int coop = a->emulated ? 0 : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  if (a->cluster_attn) {
    // co-residency: G <= the GPCs' max active clusters (llama_step_grid)
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = N;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;  // all-or-nothing residency
    at[1].val.cooperative = coop;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (p.kv_pages) {
      auto kern = a->cluster_attn == 2 ? llama_step_kernel<true, false, true> : llama_step_kernel<true, true, true>;
      if (const int rc = configure_kernel((const void*)kern, kMaxSmem, true)) return rc;
      CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
    } else if (a->cluster_attn == 2) {
      if (const int rc = configure_kernel((const void*)llama_step_kernel<true, false>, kMaxSmem, true))
        return rc;
      CFB_CUDA(cudaLaunchKernelEx(&cfg, llama_step_kernel<true, false>, p));
    } else {
      CFB_CUDA(cudaLaunchKernelEx(&cfg, llama_step_kernel<true>, p));
    }
  } else {
    if (const int rc = configure_kernel((const void*)llama_step_kernel<false>, kMaxSmem, false)) return rc;
    at[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (grid barriers)
    at[0].val.cooperative = coop;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, llama_step_kernel<false>, p));
  }
  return CFB_OK;
}

}  // namespace cfb
