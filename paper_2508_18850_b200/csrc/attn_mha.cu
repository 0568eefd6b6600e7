// split_token fused attention module (ClusterFusion Alg. 3) for sm_100a.
//
// Mirrors reference dataflows.py:235-313 (run_fused_mha_decode):
//   one cluster of N CTAs per head (grid N x n_heads), CTA rank r:
//   1. QKV GEMV over its head-dim slice [r*h, (r+1)*h) of q, k and v
//      (rows stream from HBM by TMA bulk copies)            dataflows.py:256-267
//   2. ClusterGather of the 3h-slices (DSMEM), canonical order  :268-279
//   3. (model mode) RoPE + KV-cache append of the new token
//   4. flash-decoding over KV segment [r*ceil(S/N), ...); the new token's
//      K/V join rank N-1's segment only                       :283-295
//   5. softmax-stat merge: MAX reduce, rescaled SUM reduce (or one
//      SOFTMAX_MERGE pair reduce)                             :187-227
//   6. rescale A by exp(m_b - m*)/l*, SUM reduce of A (DSMEM) :298-300
//   7. O-proj over output columns [r*D/N, (r+1)*D/N)         :302-310
//   8. cross-head sum: every CTA adds its O-proj columns into a 64-bit
//      fixed-point accumulator (value * 2^32, red.global.add.u64).  Integer
//      addition is associative, so the sum is bit-identical whatever order
//      the 32 heads' CTAs arrive in: a deterministic replacement of the
//      reference's atomic_accumulate (dataflows.py:302-310) with no tickets,
//      fences or serial tail.  The consumer (the FFN prologue in the decode
//      engine, or mha_finalize_kernel for the API) converts it back to fp32.
// Storage rounding follows simcore.py: every buffer store is rounded to T.
//
// Programmatic dependent launch: the producer warp streams this CTA's W_qkv
// rows before griddepcontrol.wait, i.e. while the previous kernel is still
// finishing; everything that reads activations, the step position or the KV
// cache happens after the wait.
#include <cuda_runtime.h>

#include "collectives.cuh"
#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct MhaParams {
  int B, D, H, Hp, N, n_heads, S_static, cache_cap, flags, spw, sleep_max;
  float inv_sqrt_h, eps;
  const void* x;
  const float* resid;
  const void* norm_w;
  const void* w_qkv;
  const void* w_out;
  void* k_cache;
  void* v_cache;
  const float* rope_cs;
  const int* step_pos;
  unsigned long long* accum;  // [B][D] fixed-point head sum (2^-32 units)
  float* stats;
  unsigned long long* traffic;
  unsigned long long* trace;
};

struct MhaLayout {
  int bars, x, part, gbuf, qf, ws_acc, ws_ml, loc, abuf, arx, st, strx, red, pay, total;
  int seg_bytes, a_bytes, st_bytes, pay_bytes;
};

__host__ __device__ inline int round16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline MhaLayout mha_layout(int B, int D, int Hp, int N, int tb, int spw,
                                                bool oneshot) {
  MhaLayout L;
  const int h = Hp / N;
  int rounds = 0;
  while ((1 << rounds) < N) ++rounds;
  L.seg_bytes = round16(B * 3 * h * tb);
  L.a_bytes = round16(B * Hp * tb);
  L.st_bytes = round16(2 * B * tb);
  L.pay_bytes = oneshot ? round16((2 * B + B * Hp) * 4) : 0;  // fp32 [m | l | A]
  int o = ring_bytes(spw);
  L.bars = o;       o += (2 * kNumSlots + 16) * 8;
  L.x = o;          o += round16(B * (D > Hp ? D : Hp) * 4);  // fp32, tile-GEMV layout
  L.part = o;       o += round16(kNumConsumerWarps * B * 3 * h * 4);
  L.gbuf = o;       o += N * L.seg_bytes;
  L.qf = o;         o += 3 * B * Hp * 4;
  L.ws_acc = o;     o += kNumConsumerWarps * B * Hp * 4;
  L.ws_ml = o;      o += kNumConsumerWarps * B * 2 * 4;
  L.loc = o;        o += round16(4 * B * 4);  // m_loc, l_loc, m_star, l_star
  L.abuf = o;       o += L.a_bytes;
  L.arx = o;        o += 4 * L.a_bytes;
  L.st = o;         o += 2 * L.st_bytes;
  L.strx = o;       o += 8 * L.st_bytes;
  L.red = o;        o += round16(kNumConsumerWarps * B * 4);
  L.pay = o;        o += N * L.pay_bytes;
  L.total = o;
  return L;
}

template <typename T, int EPL, int QB>
__global__ void __launch_bounds__(kThreads, 1) mha_split_token_kernel(const MhaParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  constexpr bool XH = sizeof(T) == 2;  // GEMV activations as fp16 in smem (FHFMA path)
  // keys per online-softmax chunk: a chunk's dot products,
  // shuffle reductions and exponentials are independent, which is the ILP
  // that hides shuffle/MUFU latency with only 8 consumer warps per SM
  constexpr int RC = QB == 1 ? 4 : (QB <= 4 ? 2 : 1);
  const int B = p.B, D = p.D, Hp = p.Hp;
  const uint32_t N = p.N;
  const int h = Hp / N;
  const bool oneshot = p.flags & CFB_ONESHOT;
  const MhaLayout L = mha_layout(B, D, Hp, N, tb, p.spw, oneshot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  uint64_t* cbar = bars + 2 * kNumSlots;  // [0,4) gather, [4,8) max/merge, [8,12) sum, [12,16) attn
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int head = blockIdx.y;
  int rounds = 0;
  while ((1u << rounds) < N) ++rounds;
  const bool merged = p.flags & CFB_STATS_MERGED;

  if (tid == 0 && oneshot) {
    ring_init(ring);
    mbar_init(&cbar[0], 1);
    mbar_arrive_expect_tx(&cbar[0], (N - 1) * L.seg_bytes);
    mbar_init(&cbar[4], 1);
    mbar_arrive_expect_tx(&cbar[4], (N - 1) * L.pay_bytes);
    fence_mbar_init();
  } else if (tid == 0) {
    ring_init(ring);
    for (int r = 0; r < rounds; ++r) {
      mbar_init(&cbar[r], 1);
      mbar_arrive_expect_tx(&cbar[r], (1u << r) * L.seg_bytes);
      mbar_init(&cbar[4 + r], 1);
      mbar_arrive_expect_tx(&cbar[4 + r], L.st_bytes);
      mbar_init(&cbar[8 + r], 1);
      mbar_arrive_expect_tx(&cbar[8 + r], L.st_bytes);
      mbar_init(&cbar[12 + r], 1);
      mbar_arrive_expect_tx(&cbar[12 + r], L.a_bytes);
    }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_arrive();
  pdl_launch_dependents();

  const size_t cache_head = (size_t)head * p.cache_cap * Hp;
  const int qkv_rows = 3 * h, qkv_tiles = (qkv_rows + kTileRows - 1) / kTileRows;
  const Phase P0 = make_phase(static_cast<const T*>(p.w_qkv) +
                                  ((size_t)head * N + rank) * qkv_tiles * kTileRows * D,
                              nullptr, qkv_tiles, kTileRows * D * tb, true);
  const int cols = D / (int)N;
  const Phase P2 = make_phase(static_cast<const T*>(p.w_out) + ((size_t)head * N + rank) * cols * Hp,
                              nullptr, cols, Hp * tb);
  auto kv_phase = [&](int S) {
    const int seg = S == 0 ? 0 : (S + (int)N - 1) / (int)N;
    const int lo = min((int)rank * seg, S), hi = min(lo + seg, S);
    return make_phase(static_cast<const T*>(p.k_cache) + cache_head + (size_t)lo * Hp,
                      static_cast<const T*>(p.v_cache) + cache_head + (size_t)lo * Hp, hi - lo,
                      Hp * tb);
  };

  if (warp == kNumConsumerWarps) {  // ------------------------------ producer
    int c = 0;
    {
      const Phase ph0[1] = {P0};
      produce_all(ph0, ring, lane, policy_evict_first(), c);  // weights: before the PDL wait
    }
    pdl_wait();
    const int S = p.step_pos ? *p.step_pos : p.S_static;
    const Phase ph1[2] = {kv_phase(S), P2};
    produce_all(ph1, ring, lane, policy_evict_first(), c);
    __syncwarp();
    cluster_wait();
    cluster_arrive();
    cluster_wait();
    return;
  }

  // ---------------------------------------------------------------- consumers
  unsigned long long* tr =
      p.trace ? p.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer();
  XElem<XH>* xs = reinterpret_cast<XElem<XH>*>(smem + L.x);
  float* part = reinterpret_cast<float*>(smem + L.part);
  T* gseg = reinterpret_cast<T*>(smem + L.gbuf);
  float* qf = reinterpret_cast<float*>(smem + L.qf);
  float* kf = qf + B * Hp;
  float* vf = kf + B * Hp;
  float* ws_acc = reinterpret_cast<float*>(smem + L.ws_acc);
  float* ws_m = reinterpret_cast<float*>(smem + L.ws_ml);
  float* ws_l = ws_m + kNumConsumerWarps * B;
  float* m_loc = reinterpret_cast<float*>(smem + L.loc);
  float* l_loc = m_loc + B;
  float* m_st = l_loc + B;
  float* l_st = m_st + B;
  T* abuf = reinterpret_cast<T*>(smem + L.abuf);
  float* red = reinterpret_cast<float*>(smem + L.red);
  unsigned long long sent[5] = {0, 0, 0, 0, 0};  // gather, max, sum, merge, attn

  pdl_wait();  // activations / step position / KV cache of the previous kernel
  const int S = p.step_pos ? *p.step_pos : p.S_static;
  const Phase P1 = kv_phase(S);

  int cnt = 0;
  // 1. activations
  if (p.flags & CFB_NORM) {
    rmsnorm_to_smem<T, XH>(xs, p.resid, static_cast<const T*>(p.norm_w), B, D, p.eps, red, tid);
  } else {
    load_act_to_smem<T, XH>(xs, static_cast<const T*>(p.x), B, D, tid);
  }

  // 2. QKV GEMV: rows of [q-slice | k-slice | v-slice] for this rank
  if (tr && tid == 0) tr[1] = globaltimer();
  tiled_gemv_phase<T, QB, XH>(P0, ring, warp, lane, tid, cnt, xs, D, B, qkv_rows, part,
                          [&](int row, int b, float v) { gseg[b * 3 * h + row] = Elem<T>::from_f(v); });
  consumer_sync();

  if (tr && tid == 0) tr[2] = globaltimer();
  cluster_wait();  // peers' mbarriers are initialised from here on
  if (tr && tid == 0) tr[8] = globaltimer();

  // 3. ClusterGather of the qkv slices
  const int seg_elems = L.seg_bytes / tb;
  if (warp == 0 && N > 1 && oneshot) {
    // one round: push the local segment into slot (peer - rank) mod N of every
    // peer (the same rank-rotated layout the log2(N)-round schedule leaves)
    for (uint32_t d = 1; d < N; ++d) {
      const uint32_t peer = (rank + d) % N;
      dsmem_push(gseg, reinterpret_cast<char*>(gseg) + d * L.seg_bytes, &cbar[0], L.seg_bytes, peer,
                 lane);
    }
    sent[0] += (unsigned long long)(N - 1) * B * 3 * (p.H / N) * tb;
    __syncwarp();
    mbar_wait(&cbar[0], 0);
  } else if (warp == 0 && N > 1) {
    uint64_t* gb[4] = {&cbar[0], &cbar[1], &cbar[2], &cbar[3]};
    warp_cluster_gather(reinterpret_cast<char*>(gseg), L.seg_bytes, gb, rank, N, lane);
    for (uint32_t s = 1; s < N; s <<= 1) sent[0] += (unsigned long long)s * B * 3 * (p.H / N) * tb;
  }
  consumer_sync();
  for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
    const int b = idx / Hp, d = idx % Hp;
    const int r = d / h, i = d % h;
    const T* sg = gseg + ((rank - r + N) % N) * seg_elems + b * 3 * h;
    qf[idx] = Elem<T>::to_f(sg[i]);
    kf[idx] = Elem<T>::to_f(sg[h + i]);
    vf[idx] = Elem<T>::to_f(sg[2 * h + i]);
  }
  consumer_sync();
  if (p.flags & CFB_ROPE) {  // RoPE (rotate-half) at position S + b
    const int half = Hp / 2;
    for (int idx = tid; idx < B * half; idx += kConsumerThreads) {
      const int b = idx / half, i = idx % half;
      const float c = p.rope_cs[((size_t)(S + b) * half + i) * 2];
      const float sn = p.rope_cs[((size_t)(S + b) * half + i) * 2 + 1];
      float* qb = qf + b * Hp;
      float* kb = kf + b * Hp;
      const float q1 = qb[i], q2 = qb[i + half], k1 = kb[i], k2 = kb[i + half];
      qb[i] = round_to<T>(__fsub_rn(__fmul_rn(q1, c), __fmul_rn(q2, sn)));
      qb[i + half] = round_to<T>(__fadd_rn(__fmul_rn(q2, c), __fmul_rn(q1, sn)));
      kb[i] = round_to<T>(__fsub_rn(__fmul_rn(k1, c), __fmul_rn(k2, sn)));
      kb[i + half] = round_to<T>(__fadd_rn(__fmul_rn(k2, c), __fmul_rn(k1, sn)));
    }
    consumer_sync();
  }
  if ((p.flags & CFB_WRITE_KV) && rank == N - 1) {  // KV-cache append at rows S..S+B-1
    T* kc = static_cast<T*>(p.k_cache) + cache_head;
    T* vc = static_cast<T*>(p.v_cache) + cache_head;
    for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
      kc[(size_t)S * Hp + idx] = Elem<T>::from_f(kf[idx]);
      vc[(size_t)S * Hp + idx] = Elem<T>::from_f(vf[idx]);
    }
  }

  if (tr && tid == 0) tr[3] = globaltimer();
  // 4. split-KV flash decoding over this rank's segment.  A warp covers KPP
  //    keys per step (LPK lanes x EPL dims each); RC steps form one chunk
  //    whose scores share one max/rescale (online softmax per chunk).
  const int LPK = Hp / EPL, KPP = 32 / LPK, g = lane / LPK, li = lane % LPK;
  const float inv_sqrt_h = p.inv_sqrt_h;
  float q[QB][EPL], acc[QB][EPL], m[QB], l[QB];
#pragma unroll
  for (int b = 0; b < QB; ++b) {
    m[b] = -INFINITY;
    l[b] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      q[b][e] = (b < B) ? qf[b * Hp + li * EPL + e] : 0.f;
      acc[b][e] = 0.f;
    }
  }
  auto attend = [&](auto&& load_k, auto&& load_v, int nkeys) {
    for (int k0 = 0; k0 < nkeys; k0 += RC * KPP) {
      float s[RC][QB];
      bool valid[RC];
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        const int key = k0 + j * KPP + g;
        valid[j] = key < nkeys;
        float kv[EPL];
        load_k(valid[j] ? key : 0, kv);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          float t = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) t = fmaf(q[b][e], kv[e], t);
          s[j][b] = t;
        }
      }
      for (int o = 1; o < LPK; o <<= 1) {
#pragma unroll
        for (int j = 0; j < RC; ++j)
#pragma unroll
          for (int b = 0; b < QB; ++b) s[j][b] += __shfl_xor_sync(0xffffffffu, s[j][b], o);
      }
      float vv[RC][EPL];
#pragma unroll
      for (int j = 0; j < RC; ++j) load_v(valid[j] ? k0 + j * KPP + g : 0, vv[j]);
#pragma unroll
      for (int b = 0; b < QB; ++b) {
        if (b >= B) continue;
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          s[j][b] = valid[j] ? __fmul_rn(s[j][b], inv_sqrt_h) : -INFINITY;
          mx = fmaxf(mx, s[j][b]);
        }
        for (int o = LPK; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float mn = fmaxf(m[b], mx);  // finite: the chunk has >= 1 valid key
        const float alpha = __expf(m[b] - mn);  // m = -inf -> 0
        float ps = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[b][e] *= alpha;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const float pr = __expf(s[j][b] - mn);  // invalid: exp(-inf) = 0
          ps += pr;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[b][e] = fmaf(pr, vv[j][e], acc[b][e]);
        }
        l[b] = fmaf(l[b], alpha, ps);
        m[b] = mn;
      }
    }
  };
  if (tr && tid == 0) tr[11] = globaltimer();
  consume_phase(P1, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    const T* K = reinterpret_cast<const T*>(slot);
    const T* V = reinterpret_cast<const T*>(slot + kSlotBytes / 2);
    attend([&](int k, float* o) { load_elems<T, EPL>(K + k * Hp + li * EPL, o); },
           [&](int k, float* o) { load_elems<T, EPL>(V + k * Hp + li * EPL, o); }, it.nunits);
  });
  if (tr && tid == 0) tr[12] = globaltimer();
  if ((p.flags & CFB_APPEND) && rank == N - 1 && warp == 0) {  // new token(s): counted once
    attend([&](int k, float* o) {
             for (int e = 0; e < EPL; ++e) o[e] = kf[k * Hp + li * EPL + e];
           },
           [&](int k, float* o) {
             for (int e = 0; e < EPL; ++e) o[e] = vf[k * Hp + li * EPL + e];
           },
           B);
  }
  // fold the KPP key groups of the warp (same lane-in-group = same dims);
  // the groups share m (warp-uniform), so l and acc simply add
#pragma unroll
  for (int b = 0; b < QB; ++b) {
    for (int o = LPK; o < 32; o <<= 1) {
      l[b] += __shfl_xor_sync(0xffffffffu, l[b], o);
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[b][e] += __shfl_xor_sync(0xffffffffu, acc[b][e], o);
    }
    if (b < B) {
      if (g == 0) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) ws_acc[(warp * B + b) * Hp + li * EPL + e] = acc[b][e];
      }
      if (lane == 0) {
        ws_m[warp * B + b] = m[b];
        ws_l[warp * B + b] = l[b];
      }
    }
  }
  consumer_sync();
  if (tr && tid == 0) tr[13] = globaltimer();
  // merge the 8 warp states in warp order -> (A_loc, m_loc, l_loc); every
  // thread recomputes the (cheap) per-warp factors of its batch row, so the
  // merge is one parallel pass with no serial section
  const int pw = L.pay_bytes / 4;
  float* pay = reinterpret_cast<float*>(smem + L.pay);
  float* mine = pay + rank * pw;  // oneshot: fp32 exchange payload [m | l | A]
  for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
    const int b = idx / Hp;
    float mm = -INFINITY;
#pragma unroll
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) mm = fmaxf(mm, ws_m[w2 * B + b]);
    float ll = 0.f, a = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) {
      const float mw = ws_m[w2 * B + b];
      const float f = (mw == -INFINITY) ? 0.f : expf(mw - mm);
      ll = fmaf(ws_l[w2 * B + b], f, ll);
      a = fmaf(ws_acc[(w2 * B + b) * Hp + idx % Hp], f, a);
    }
    if (oneshot) {
      mine[2 * B + idx] = a;
    } else {
      abuf[idx] = Elem<T>::from_f(a);  // block.store("attn_out", a_part)
    }
    if (idx % Hp == 0) {
      m_loc[b] = mm;
      l_loc[b] = ll;
      if (oneshot) {
        mine[b] = mm;
        mine[B + b] = ll;
      }
    }
  }
  if (!oneshot)
    for (int idx = B * Hp + tid; idx < L.a_bytes / tb; idx += kConsumerThreads)
      abuf[idx] = Elem<T>::from_f(0.f);
  consumer_sync();
  if (oneshot) {
    // Fused statistics + attention-output exchange in ONE round: every CTA
    // pushes its fp32 partial state (m_loc, l_loc, unnormalised A_loc) into
    // slot `rank` of every peer, then all CTAs merge the N states in rank
    // order (identical, deterministic result everywhere):
    //   m* = max_r m_r,  l* = sum_r l_r e^{m_r - m*},  A* = sum_r A_r e^{m_r - m*} / l*
    // = the reference's MAX-reduce / rescale / SUM-reduce / rescale / SUM-reduce
    // sequence (dataflows.py:187-232, :297-300) with all partial stores in fp32.
    if (tr && tid == 0) tr[4] = globaltimer();
    if (warp == 0 && N > 1) {
      for (uint32_t d = 1; d < N; ++d)
        dsmem_push(mine, mine, &cbar[4], L.pay_bytes, (rank + d) % N, lane);
      sent[4] += (unsigned long long)(N - 1) * (2 * B + B * p.H) * 4;
    }
    if (tr && tid == 0) tr[9] = globaltimer();
    if (N > 1) mbar_wait(&cbar[4], 0);
    if (tr && tid == 0) tr[10] = globaltimer();
    for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
      const int b = idx / Hp;
      float ms = -INFINITY;
      for (uint32_t r = 0; r < N; ++r) ms = fmaxf(ms, pay[r * pw + b]);
      float ls = 0.f, a = 0.f;
      for (uint32_t r = 0; r < N; ++r) {
        const float mr = pay[r * pw + b];
        const float f = (mr == -INFINITY) ? 0.f : expf(mr - ms);
        ls = fmaf(pay[r * pw + B + b], f, ls);
        a = fmaf(pay[r * pw + 2 * B + idx], f, a);
      }
      abuf[idx] = Elem<T>::from_f(__fdiv_rn(a, ls));
      if (idx % Hp == 0) {
        m_st[b] = ms;
        l_st[b] = ls;
      }
    }
    consumer_sync();
    if (warp == 0) {
      if (rank == 0 && p.stats)
        for (int b = lane; b < B; b += 32) {
          p.stats[((size_t)head * 2) * B + b] = m_st[b];
          p.stats[((size_t)head * 2 + 1) * B + b] = l_st[b];
        }
      if (lane == 0 && p.traffic) {
        atomicAdd(&p.traffic[0], sent[0]);
        atomicAdd(&p.traffic[4], sent[4]);
      }
    }
  } else {

    if (tr && tid == 0) tr[4] = globaltimer();
    // 5. softmax statistics
    T* st0 = reinterpret_cast<T*>(smem + L.st);
    T* st1 = reinterpret_cast<T*>(smem + L.st + L.st_bytes);
    if (warp == 0) {
      T* rx[4];
      uint64_t* rb[4];
      for (int i = lane; i < L.st_bytes / tb; i += 32) {
        st0[i] = Elem<T>::from_f(0.f);
        st1[i] = Elem<T>::from_f(0.f);
      }
      __syncwarp();
      if (merged) {
        for (int b = lane; b < B; b += 32) {
          st0[b] = Elem<T>::from_f(m_loc[b]);
          st0[B + b] = Elem<T>::from_f(l_loc[b]);
        }
        __syncwarp();
        for (int r = 0; r < 4; ++r) {
          rx[r] = reinterpret_cast<T*>(smem + L.strx + r * L.st_bytes);
          rb[r] = &cbar[4 + r];
        }
        warp_cluster_reduce<T>(st0, 2 * B, L.st_bytes, rx, rb, kSoftmaxMerge, rank, N, lane);
        for (int r = 0; r < rounds; ++r) sent[3] += 2ull * B * tb;
        for (int b = lane; b < B; b += 32) {
          m_st[b] = Elem<T>::to_f(st0[b]);
          l_st[b] = Elem<T>::to_f(st0[B + b]);
        }
      } else {
        for (int b = lane; b < B; b += 32) st0[b] = Elem<T>::from_f(m_loc[b]);
        __syncwarp();
        for (int r = 0; r < 4; ++r) {
          rx[r] = reinterpret_cast<T*>(smem + L.strx + r * L.st_bytes);
          rb[r] = &cbar[4 + r];
        }
        warp_cluster_reduce<T>(st0, B, L.st_bytes, rx, rb, kMax, rank, N, lane);
        for (int b = lane; b < B; b += 32) {
          const float ms = Elem<T>::to_f(st0[b]);
          m_st[b] = ms;
          const float f = (m_loc[b] == -INFINITY) ? 0.f : expf(m_loc[b] - ms);
          st1[b] = Elem<T>::from_f(__fmul_rn(l_loc[b], f));
        }
        __syncwarp();
        for (int r = 0; r < 4; ++r) {
          rx[r] = reinterpret_cast<T*>(smem + L.strx + (4 + r) * L.st_bytes);
          rb[r] = &cbar[8 + r];
        }
        warp_cluster_reduce<T>(st1, B, L.st_bytes, rx, rb, kSum, rank, N, lane);
        for (int b = lane; b < B; b += 32) l_st[b] = Elem<T>::to_f(st1[b]);
        for (int r = 0; r < rounds; ++r) {
          sent[1] += (unsigned long long)B * tb;
          sent[2] += (unsigned long long)B * tb;
        }
      }
    }
    consumer_sync();
    // 6. rescale and reduce the attention output
    for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
      const int b = idx / Hp;
      const float e = (m_loc[b] == -INFINITY) ? 0.f : expf(m_loc[b] - m_st[b]);
      const float f = __fdiv_rn(e, l_st[b]);
      abuf[idx] = Elem<T>::from_f(__fmul_rn(Elem<T>::to_f(abuf[idx]), f));
    }
    consumer_sync();
    if (warp == 0) {
      T* rx[4];
      uint64_t* rb[4];
      for (int r = 0; r < 4; ++r) {
        rx[r] = reinterpret_cast<T*>(smem + L.arx + r * L.a_bytes);
        rb[r] = &cbar[12 + r];
      }
      warp_cluster_reduce<T>(abuf, B * Hp, L.a_bytes, rx, rb, kSum, rank, N, lane);
      for (int r = 0; r < rounds; ++r) sent[4] += (unsigned long long)B * p.H * tb;
      if (rank == 0 && p.stats)
        for (int b = lane; b < B; b += 32) {
          p.stats[((size_t)head * 2) * B + b] = m_st[b];
          p.stats[((size_t)head * 2 + 1) * B + b] = l_st[b];
        }
      if (lane == 0 && p.traffic) {
        atomicAdd(&p.traffic[0], sent[0]);
        if (merged) {
          atomicAdd(&p.traffic[3], sent[3]);
        } else {
          atomicAdd(&p.traffic[1], sent[1]);
          atomicAdd(&p.traffic[2], sent[2]);
        }
        atomicAdd(&p.traffic[4], sent[4]);
      }
    }
    consumer_sync();
  }
  if (tr && tid == 0) tr[5] = globaltimer();
  // 7. O-projection over this rank's output columns (row-tiled W_out^T slice,
  //    the same conflict-free tile GEMV as the QKV phase, K = head_pad) and
  // 8. the cross-head sum into the fixed-point accumulator
  const int c_base = (int)rank * cols;
  long long cyc_math = 0, nitems = 0;
  consume_phase(P2, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    const long long c0 = clock64();
    ++nitems;
    rowlane_item<T, QB>(it, slot, abuf, Hp, B, lane, [&](int row, const float (&s)[QB]) {
#pragma unroll
      for (int b = 0; b < QB; ++b)
        if (b < B) red_add_fixed(&p.accum[(size_t)b * D + c_base + row], s[b]);
    });
    cyc_math += clock64() - c0;
  });
  if (tr && tid == 0) {
    tr[6] = globaltimer();
    tr[14] = cyc_math;
    tr[15] = nitems;
  }
  cluster_arrive();
  cluster_wait();
  if (tr && tid == 0) tr[7] = globaltimer();
}

// API epilogue: out = [resid +] accum * 2^-32, then re-zero the accumulator.
__global__ void mha_finalize_kernel(float* out, const float* resid,
                                    unsigned long long* accum, int n) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float v = fixed_to_float(accum[i]);
    out[i] = resid ? __fadd_rn(resid[i], v) : v;
    accum[i] = 0ull;
  }
}

// ---------------------------------------------------------------- host side

template <typename T, int EPL, int QB>
static int launch_mha_inst(const MhaParams& p, size_t smem, cudaStream_t st, bool pdl) {
  auto kern = mha_split_token_kernel<T, EPL, QB>;
  if (const int rc = configure_kernel((const void*)kern, kMaxSmem, true)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.N, p.n_heads, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  LaunchAttrs at(p.N, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

template <typename T>
static int launch_mha_t(const MhaParams& p, size_t smem, cudaStream_t st, bool pdl) {
  if (p.B > 4) return launch_mha_inst<T, 4, 16>(p, smem, st, pdl);
  if (p.Hp == 8) {  // EPL: attention elements per lane
    if (p.B == 1) return launch_mha_inst<T, 8, 1>(p, smem, st, pdl);
    if (p.B == 2) return launch_mha_inst<T, 8, 2>(p, smem, st, pdl);
    return launch_mha_inst<T, 8, 4>(p, smem, st, pdl);
  }
  if (p.B == 1) return launch_mha_inst<T, 16, 1>(p, smem, st, pdl);
  if (p.B == 2) return launch_mha_inst<T, 16, 2>(p, smem, st, pdl);
  return launch_mha_inst<T, 16, 4>(p, smem, st, pdl);
}

int mha_decode(const cfb_mha_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->dtype != CFB_F16 && a->dtype != CFB_F32)
    return set_error(CFB_ERR_ARGUMENT, "dtype must be CFB_F16 (2) or CFB_F32 (4)");
  const int N = a->cluster, tb = a->dtype;
  if (N < 1 || N > 16 || (N & (N - 1)))
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16], got %d", N);
  if (a->batch < 1 || a->batch > 16) return set_error(CFB_ERR_DIMENSION, "batch must be in [1, 16]");
  const int Hp = a->head_pad;
  if (Hp < 8 || (Hp & (Hp - 1)) || Hp < a->head_dim || Hp > 512)
    return set_error(CFB_ERR_DIMENSION, "head_pad must be a power of two in [8, 512] >= head_dim");
  if (a->batch > 4 && Hp > 128)
    return set_error(CFB_ERR_DIMENSION, "batch > 4 requires head_pad <= 128");
  if (Hp % N || a->head_dim % N)
    return set_error(CFB_ERR_DIMENSION, "head_dim %d not divisible by cluster size %d", a->head_dim, N);
  if (a->hidden % N || (a->hidden * tb) % 16 || ((a->hidden / N) < 1))
    return set_error(CFB_ERR_DIMENSION, "hidden %d must be divisible by cluster size and 16-byte rows",
                     a->hidden);
  if (!a->step_pos && a->seq_len < 0) return set_error(CFB_ERR_DIMENSION, "seq_len must be >= 0");
  if (!a->step_pos && a->seq_len == 0 && !(a->flags & CFB_APPEND))
    return set_error(CFB_ERR_DIMENSION, "no attended positions: empty cache and no appended token");
  if ((a->flags & CFB_ROPE) && (!a->rope_cs || Hp != a->head_dim))
    return set_error(CFB_ERR_ARGUMENT, "CFB_ROPE needs rope_cs and head_pad == head_dim");
  if ((a->flags & (CFB_NORM | CFB_RESID)) && !a->resid)
    return set_error(CFB_ERR_ARGUMENT, "CFB_NORM/CFB_RESID need resid");
  if ((a->flags & CFB_NORM) && !a->norm_w) return set_error(CFB_ERR_ARGUMENT, "CFB_NORM needs norm_w");
  if (!(a->flags & CFB_NORM) && !a->x) return set_error(CFB_ERR_ARGUMENT, "x is null");
  if (!a->w_qkv || !a->w_out || !a->k_cache || !a->v_cache || !a->accum)
    return set_error(CFB_ERR_ARGUMENT, "null weight / cache / accumulator pointer");
  int spw = tuned_spw();
  const bool oneshot = a->flags & CFB_ONESHOT;
  MhaLayout L = mha_layout(a->batch, a->hidden, Hp, N, tb, spw, oneshot);
  while (L.total > kMaxSmem && spw > 1) L = mha_layout(a->batch, a->hidden, Hp, N, tb, --spw, oneshot);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "split_token schedule needs %d B of shared memory per CTA (max %d)",
                     L.total, kMaxSmem);
  MhaParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.H = a->head_dim;
  p.Hp = Hp;
  p.N = N;
  p.n_heads = a->n_heads;
  p.S_static = a->seq_len;
  p.cache_cap = a->cache_cap;
  p.flags = a->flags;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.inv_sqrt_h = (float)(1.0 / std::sqrt((double)a->head_dim));
  p.eps = a->eps;
  p.x = a->x;
  p.resid = a->resid;
  p.norm_w = a->norm_w;
  p.w_qkv = a->w_qkv;
  p.w_out = a->w_out;
  p.k_cache = a->k_cache;
  p.v_cache = a->v_cache;
  p.rope_cs = a->rope_cs;
  p.step_pos = a->step_pos;
  p.accum = a->accum;
  p.stats = a->stats;
  p.traffic = a->traffic;
  p.trace = a->trace;
  const bool pdl = a->flags & CFB_PDL;
  int rc = tb == 2 ? launch_mha_t<__half>(p, L.total, st, pdl) : launch_mha_t<float>(p, L.total, st, pdl);
  if (rc || !a->out) return rc;
  return mha_finalize(a->out, (a->flags & CFB_RESID) ? a->resid : nullptr, a->accum,
                      a->batch * a->hidden, st);
}

int mha_finalize(float* out, const float* resid, unsigned long long* accum, int n, cudaStream_t st) {
  mha_finalize_kernel<<<(n + 255) / 256, 256, 0, st>>>(out, resid, accum, n);
  CFB_CUDA(cudaGetLastError());
  return CFB_OK;
}

}  // namespace cfb
