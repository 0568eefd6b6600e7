// fused_mla latent-attention module (ClusterFusion App. B.1) for sm_100a.
//
// Mirrors reference dataflows.py:316-429 (run_fused_mla_decode): one
// cluster of N CTAs per head (grid N x n_heads), CTA rank r:
//   1. q-proj GEMV over head-dim slice r*h..  (h = H/N) and the latent
//      down-projection GEMV over kv_lora slice r*rs.. (rs = R/N); both
//      stream row tiles of [W_q[head] | W_kv] by TMA bulk copies
//                                               dataflows.py:336-368
//   2. ClusterGather of the q slices -> q (B x H); ClusterGather of the latent
//      slices -> the new token's latent row (B x R)          :340-368
//   3. absorbed query slice q @ W_up[head][:, r*rs..] (row-per-lane GEMV over
//      K = H), ClusterGather -> q_lat (B x R)                :370-386
//   4. flash-decoding over latent-cache segment r (K = V = latent rows,
//      scale 1/sqrt(R)); the new latent rows join rank N-1 only  :388-399
//   5. softmax statistics (two_pass / merged) and SUM reduce of the
//      rescaled attention output z (B x R)                   :401-404
//   6. down-projection partial z[:, r-slice] @ W_down[head][r-slice, :]
//      (row-per-lane over K = rs), SUM reduce (B x H)        :408-416
//   7. O-projection over output columns r*D/N.. (row-per-lane, K = H) into
//      the 64-bit fixed-point cross-head accumulator        :418-425
// Every buffer store is rounded to T (simcore.py:94-110).  W_kv and the
// latent cache are shared by all heads (one HBM copy, L2-resident reuse).
#include <cuda_runtime.h>

#include "collectives.cuh"
#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct MlaParams {
  int B, D, H, Hp, R, Rp, rsp, N, n_heads, S, flags, spw, sleep_max;
  float inv_sqrt_r, eps;
  const void* x;
  const float* resid;   // [B][D] fp32 (CFB_NORM)
  const void* norm_w;   // [D] T (CFB_NORM)
  const void* w_q;    // [head][rank][tiles of h rows][D] row tiles
  const void* w_kv;   // [rank][tiles of rs rows][D] row tiles
  const void* w_up;   // [head][rank][rs rows][Hp] chunk-rotated (W_up^T slice)
  const void* w_down; // [head][rank][Hp rows][rsp] chunk-rotated (W_down^T slice)
  const void* w_out;  // [head][rank][D/N rows][Hp] chunk-rotated
  const void* cache;  // [cap][Rp] latent cache
  unsigned long long* accum;
  float* stats;
  unsigned long long* traffic;
};

struct MlaLayout {
  int bars, x, part, gq, gl, gu, qv, lat, ql, ws_acc, ws_ml, loc, abuf, arx, st, strx, zs, dbuf,
      drx, red, total;
  int sq, sl, su, a_bytes, st_bytes, d_bytes;
};

__host__ __device__ inline int r16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline MlaLayout mla_layout(int B, int D, int Hp, int Rp, int rsp, int N, int h,
                                                int rs, int tb, int spw) {
  MlaLayout L;
  L.sq = r16(B * h * tb);
  L.sl = r16(B * rs * tb);
  L.su = r16(B * rs * tb);
  L.a_bytes = r16(B * Rp * tb);
  L.st_bytes = r16(2 * B * tb);
  L.d_bytes = r16(B * Hp * tb);
  const int rows0 = 4 * ((h + 3) / 4) > 4 * ((rs + 3) / 4) ? 4 * ((h + 3) / 4) : 4 * ((rs + 3) / 4);
  int o = ring_bytes(spw);
  L.bars = o;   o += (2 * kNumSlots + 32) * 8;
  L.x = o;      o += r16(B * D * 4);
  L.part = o;   o += r16(kNumConsumerWarps * B * rows0 * 4);
  L.gq = o;     o += N * L.sq;
  L.gl = o;     o += N * L.sl;
  L.gu = o;     o += N * L.su;
  L.qv = o;     o += r16(B * Hp * tb);       // q_full (T) for the W_up GEMV
  L.lat = o;    o += r16(B * Rp * 4);        // new latent rows (fp32)
  L.ql = o;     o += r16(B * Rp * 4);        // q_lat (fp32)
  L.ws_acc = o; o += kNumConsumerWarps * B * Rp * 4;
  L.ws_ml = o;  o += kNumConsumerWarps * B * 2 * 4;
  L.loc = o;    o += r16(4 * B * 4);
  L.abuf = o;   o += L.a_bytes;
  L.arx = o;    o += 4 * L.a_bytes;
  L.st = o;     o += 2 * L.st_bytes;
  L.strx = o;   o += 8 * L.st_bytes;
  L.zs = o;     o += r16(B * rsp * tb);      // z slice (T) for the W_down GEMV
  L.dbuf = o;   o += L.d_bytes;
  L.drx = o;    o += 4 * L.d_bytes;
  L.red = o;    o += r16(kNumConsumerWarps * B * 4);
  L.total = o;
  return L;
}

template <typename T, int EPL, int QB>
__global__ void __launch_bounds__(kThreads, 1) mla_fused_kernel(const MlaParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  constexpr bool XH = sizeof(T) == 2;
  constexpr int RC = QB == 1 ? 4 : (QB <= 2 ? 2 : 1);
  const int B = p.B, D = p.D, Hp = p.Hp, Rp = p.Rp;
  const uint32_t N = p.N;
  const int h = p.H / (int)N, rs = p.R / (int)N;
  const MlaLayout L = mla_layout(B, D, Hp, Rp, p.rsp, N, h, rs, tb, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  // [0,4) q gather, [4,8) latent gather, [8,12) q_lat gather, [12,16) max/merge,
  // [16,20) sum, [20,24) attn_out, [24,28) down
  uint64_t* cbar = bars + 2 * kNumSlots;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int head = blockIdx.y;
  int rounds = 0;
  while ((1u << rounds) < N) ++rounds;
  const bool merged = p.flags & CFB_STATS_MERGED;

  if (tid == 0) {
    ring_init(ring);
    for (int r = 0; r < rounds; ++r) {
      const uint32_t seg_of[3] = {(uint32_t)L.sq, (uint32_t)L.sl, (uint32_t)L.su};
      for (int g = 0; g < 3; ++g) {
        mbar_init(&cbar[4 * g + r], 1);
        mbar_arrive_expect_tx(&cbar[4 * g + r], (1u << r) * seg_of[g]);
      }
      mbar_init(&cbar[12 + r], 1);
      mbar_arrive_expect_tx(&cbar[12 + r], L.st_bytes);
      mbar_init(&cbar[16 + r], 1);
      mbar_arrive_expect_tx(&cbar[16 + r], L.st_bytes);
      mbar_init(&cbar[20 + r], 1);
      mbar_arrive_expect_tx(&cbar[20 + r], L.a_bytes);
      mbar_init(&cbar[24 + r], 1);
      mbar_arrive_expect_tx(&cbar[24 + r], L.d_bytes);
    }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_arrive();
  pdl_launch_dependents();

  const int S = p.S;
  const int seg = S == 0 ? 0 : (S + (int)N - 1) / (int)N;
  const int lo = min((int)rank * seg, S), hi = min(lo + seg, S);
  const int qt = (h + 3) / 4, lt = (rs + 3) / 4, cols = D / (int)N;
  const Phase P0 = make_phase(static_cast<const T*>(p.w_q) + ((size_t)head * N + rank) * qt * 4 * D,
                              nullptr, qt, 4 * D * tb, true);
  const Phase P0b = make_phase(static_cast<const T*>(p.w_kv) + (size_t)rank * lt * 4 * D, nullptr, lt,
                               4 * D * tb, true);
  const Phase P1 = make_phase(static_cast<const T*>(p.w_up) + ((size_t)head * N + rank) * rs * Hp,
                              nullptr, rs, Hp * tb);
  const Phase P2 = make_phase(static_cast<const T*>(p.cache) + (size_t)lo * Rp, nullptr, hi - lo,
                              Rp * tb);
  const Phase P3 = make_phase(static_cast<const T*>(p.w_down) + ((size_t)head * N + rank) * Hp * p.rsp,
                              nullptr, Hp, p.rsp * tb);
  const Phase P4 = make_phase(static_cast<const T*>(p.w_out) + ((size_t)head * N + rank) * cols * Hp,
                              nullptr, cols, Hp * tb);

  if (warp == kNumConsumerWarps) {  // ------------------------------ producer
    const Phase ph[6] = {P0, P0b, P1, P2, P3, P4};
    produce_all(ph, ring, lane, policy_evict_first());
    __syncwarp();
    cluster_wait();
    cluster_arrive();
    cluster_wait();
    return;
  }

  XElem<XH>* xs = reinterpret_cast<XElem<XH>*>(smem + L.x);
  float* part = reinterpret_cast<float*>(smem + L.part);
  T* gq = reinterpret_cast<T*>(smem + L.gq);
  T* gl = reinterpret_cast<T*>(smem + L.gl);
  T* gu = reinterpret_cast<T*>(smem + L.gu);
  T* qv = reinterpret_cast<T*>(smem + L.qv);
  float* lat = reinterpret_cast<float*>(smem + L.lat);
  float* ql = reinterpret_cast<float*>(smem + L.ql);
  float* ws_acc = reinterpret_cast<float*>(smem + L.ws_acc);
  float* ws_m = reinterpret_cast<float*>(smem + L.ws_ml);
  float* ws_l = ws_m + kNumConsumerWarps * B;
  float* m_loc = reinterpret_cast<float*>(smem + L.loc);
  float* l_loc = m_loc + B;
  float* m_st = l_loc + B;
  float* l_st = m_st + B;
  T* abuf = reinterpret_cast<T*>(smem + L.abuf);
  T* zs = reinterpret_cast<T*>(smem + L.zs);
  T* dbuf = reinterpret_cast<T*>(smem + L.dbuf);
  unsigned long long sent[CFB_STAGE_COUNT] = {};  // logical DSMEM bytes per cfb_stage

  pdl_wait();  // activations come from the stream predecessor (PDL)
  if (p.flags & CFB_NORM)
    rmsnorm_to_smem<T, XH>(xs, p.resid, static_cast<const T*>(p.norm_w), B, D, p.eps,
                           reinterpret_cast<float*>(smem + L.red), tid);
  else
    load_act_to_smem<T, XH>(xs, static_cast<const T*>(p.x), B, D, tid);

  // 1. q-proj and latent down-projection slices
  int cnt = 0;
  tiled_gemv_phase<T, QB, XH>(P0, ring, warp, lane, tid, cnt, xs, D, B, h, part,
                              [&](int row, int b, float v) { gq[b * h + row] = Elem<T>::from_f(v); });
  consumer_sync();
  tiled_gemv_phase<T, QB, XH>(P0b, ring, warp, lane, tid, cnt, xs, D, B, rs, part,
                              [&](int row, int b, float v) { gl[b * rs + row] = Elem<T>::from_f(v); });
  consumer_sync();
  cluster_wait();  // peers' mbarriers are initialised from here on

  // 2. ClusterGathers of q and of the new latent rows
  auto gather = [&](T* buf, int seg_bytes, int bar0, int payload, int stage) {
    if (warp == 0 && N > 1) {
      uint64_t* gb[4] = {&cbar[bar0], &cbar[bar0 + 1], &cbar[bar0 + 2], &cbar[bar0 + 3]};
      warp_cluster_gather(reinterpret_cast<char*>(buf), seg_bytes, gb, rank, N, lane);
      for (uint32_t s = 1; s < N; s <<= 1) sent[stage] += (unsigned long long)s * payload;
    }
    consumer_sync();
  };
  gather(gq, L.sq, 0, B * h * tb, CFB_STAGE_Q_PROJ_GATHER);
  gather(gl, L.sl, 4, B * rs * tb, CFB_STAGE_LATENT_GATHER);
  for (int idx = tid; idx < B * Hp; idx += kConsumerThreads) {
    const int b = idx / Hp, d = idx % Hp;
    T v = Elem<T>::from_f(0.f);
    if (d < p.H) {
      const int r = d / h, i = d % h;
      v = gq[((rank - r + N) % N) * (L.sq / tb) + b * h + i];
    }
    qv[idx] = v;
  }
  for (int idx = tid; idx < B * Rp; idx += kConsumerThreads) {
    const int b = idx / Rp, d = idx % Rp;
    float v = 0.f;
    if (d < p.R) {
      const int r = d / rs, i = d % rs;
      v = Elem<T>::to_f(gl[((rank - r + N) % N) * (L.sl / tb) + b * rs + i]);
    }
    lat[idx] = v;
  }
  consumer_sync();

  // 3. absorbed query slice: q @ W_up[head][:, r*rs ..]  (K = H)
  consume_phase(P1, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    rowlane_item<T, QB>(it, slot, qv, Hp, B, lane, [&](int row, const float (&s)[QB]) {
#pragma unroll
      for (int b = 0; b < QB; ++b)
        if (b < B) gu[b * rs + row] = Elem<T>::from_f(s[b]);
    });
  });
  consumer_sync();
  gather(gu, L.su, 8, B * rs * tb, CFB_STAGE_ABSORBED_Q_GATHER);
  for (int idx = tid; idx < B * Rp; idx += kConsumerThreads) {
    const int b = idx / Rp, d = idx % Rp;
    float v = 0.f;
    if (d < p.R) {
      const int r = d / rs, i = d % rs;
      v = Elem<T>::to_f(gu[((rank - r + N) % N) * (L.su / tb) + b * rs + i]);
    }
    ql[idx] = v;
  }
  consumer_sync();

  // 4. flash decoding over the latent segment (K = V)
  const int LPK = Rp / EPL, KPP = 32 / LPK, g = lane / LPK, li = lane % LPK;
  const float scale = p.inv_sqrt_r;
  float q[QB][EPL], acc[QB][EPL], m[QB], l[QB];
#pragma unroll
  for (int b = 0; b < QB; ++b) {
    m[b] = -INFINITY;
    l[b] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      q[b][e] = (b < B) ? ql[b * Rp + li * EPL + e] : 0.f;
      acc[b][e] = 0.f;
    }
  }
  auto attend = [&](auto&& load_k, int nkeys) {
    for (int k0 = 0; k0 < nkeys; k0 += RC * KPP) {
      float s[RC][QB], kv[RC][EPL];
      bool valid[RC];
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        const int key = k0 + j * KPP + g;
        valid[j] = key < nkeys;
        load_k(valid[j] ? key : 0, kv[j]);
#pragma unroll
        for (int b = 0; b < QB; ++b) {
          float t = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) t = fmaf(q[b][e], kv[j][e], t);
          s[j][b] = t;
        }
      }
      for (int o = 1; o < LPK; o <<= 1) {
#pragma unroll
        for (int j = 0; j < RC; ++j)
#pragma unroll
          for (int b = 0; b < QB; ++b) s[j][b] += __shfl_xor_sync(0xffffffffu, s[j][b], o);
      }
#pragma unroll
      for (int b = 0; b < QB; ++b) {
        if (b >= B) continue;
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          s[j][b] = valid[j] ? __fmul_rn(s[j][b], scale) : -INFINITY;
          mx = fmaxf(mx, s[j][b]);
        }
        for (int o = LPK; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float mn = fmaxf(m[b], mx);
        const float alpha = __expf(m[b] - mn);
        float ps = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[b][e] *= alpha;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const float pr = __expf(s[j][b] - mn);
          ps += pr;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[b][e] = fmaf(pr, kv[j][e], acc[b][e]);
        }
        l[b] = fmaf(l[b], alpha, ps);
        m[b] = mn;
      }
    }
  };
  consume_phase(P2, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    const T* K = reinterpret_cast<const T*>(slot);
    attend([&](int k, float* o) { load_elems<T, EPL>(K + k * Rp + li * EPL, o); }, it.nunits);
  });
  if ((p.flags & CFB_APPEND) && rank == N - 1 && warp == 0) {  // new latent rows: counted once
    attend([&](int k, float* o) {
      for (int e = 0; e < EPL; ++e) o[e] = lat[k * Rp + li * EPL + e];
    }, B);
  }
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
        for (int e = 0; e < EPL; ++e) ws_acc[(warp * B + b) * Rp + li * EPL + e] = acc[b][e];
      }
      if (lane == 0) {
        ws_m[warp * B + b] = m[b];
        ws_l[warp * B + b] = l[b];
      }
    }
  }
  consumer_sync();
  for (int idx = tid; idx < B * Rp; idx += kConsumerThreads) {
    const int b = idx / Rp;
    float mm = -INFINITY;
#pragma unroll
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) mm = fmaxf(mm, ws_m[w2 * B + b]);
    float ll = 0.f, a = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < kNumConsumerWarps; ++w2) {
      const float mw = ws_m[w2 * B + b];
      const float f = (mw == -INFINITY) ? 0.f : expf(mw - mm);
      ll = fmaf(ws_l[w2 * B + b], f, ll);
      a = fmaf(ws_acc[(w2 * B + b) * Rp + idx % Rp], f, a);
    }
    abuf[idx] = Elem<T>::from_f(a);  // block.store("attn_out", a_part)
    if (idx % Rp == 0) {
      m_loc[b] = mm;
      l_loc[b] = ll;
    }
  }
  for (int idx = B * Rp + tid; idx < L.a_bytes / tb; idx += kConsumerThreads)
    abuf[idx] = Elem<T>::from_f(0.f);
  consumer_sync();

  // 5. softmax statistics + rescaled SUM reduce of z
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
        rb[r] = &cbar[12 + r];
      }
      warp_cluster_reduce<T>(st0, 2 * B, L.st_bytes, rx, rb, kSoftmaxMerge, rank, N, lane);
      for (int r = 0; r < rounds; ++r) sent[CFB_STAGE_STATS_MERGE] += 2ull * B * tb;
      for (int b = lane; b < B; b += 32) {
        m_st[b] = Elem<T>::to_f(st0[b]);
        l_st[b] = Elem<T>::to_f(st0[B + b]);
      }
    } else {
      for (int b = lane; b < B; b += 32) st0[b] = Elem<T>::from_f(m_loc[b]);
      __syncwarp();
      for (int r = 0; r < 4; ++r) {
        rx[r] = reinterpret_cast<T*>(smem + L.strx + r * L.st_bytes);
        rb[r] = &cbar[12 + r];
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
        rb[r] = &cbar[16 + r];
      }
      warp_cluster_reduce<T>(st1, B, L.st_bytes, rx, rb, kSum, rank, N, lane);
      for (int b = lane; b < B; b += 32) l_st[b] = Elem<T>::to_f(st1[b]);
      for (int r = 0; r < rounds; ++r) {
        sent[CFB_STAGE_STATS_MAX] += (unsigned long long)B * tb;
        sent[CFB_STAGE_STATS_SUM] += (unsigned long long)B * tb;
      }
    }
  }
  consumer_sync();
  for (int idx = tid; idx < B * Rp; idx += kConsumerThreads) {
    const int b = idx / Rp;
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
      rb[r] = &cbar[20 + r];
    }
    warp_cluster_reduce<T>(abuf, B * Rp, L.a_bytes, rx, rb, kSum, rank, N, lane);
    for (int r = 0; r < rounds; ++r) sent[CFB_STAGE_ATTN_OUT] += (unsigned long long)B * p.R * tb;
    if (rank == 0 && p.stats)
      for (int b = lane; b < B; b += 32) {
        p.stats[((size_t)head * 2) * B + b] = m_st[b];
        p.stats[((size_t)head * 2 + 1) * B + b] = l_st[b];
      }
  }
  consumer_sync();

  // 6. down-projection partial over this rank's latent slice, SUM reduce
  for (int idx = tid; idx < B * p.rsp; idx += kConsumerThreads) {
    const int b = idx / p.rsp, i = idx % p.rsp;
    zs[idx] = i < rs ? abuf[b * Rp + rank * rs + i] : Elem<T>::from_f(0.f);
  }
  for (int idx = tid; idx < L.d_bytes / tb; idx += kConsumerThreads) dbuf[idx] = Elem<T>::from_f(0.f);
  consumer_sync();
  consume_phase(P3, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    rowlane_item<T, QB>(it, slot, zs, p.rsp, B, lane, [&](int row, const float (&s)[QB]) {
#pragma unroll
      for (int b = 0; b < QB; ++b)
        if (b < B) dbuf[b * Hp + row] = Elem<T>::from_f(s[b]);
    });
  });
  consumer_sync();
  if (warp == 0) {
    T* rx[4];
    uint64_t* rb[4];
    for (int r = 0; r < 4; ++r) {
      rx[r] = reinterpret_cast<T*>(smem + L.drx + r * L.d_bytes);
      rb[r] = &cbar[24 + r];
    }
    warp_cluster_reduce<T>(dbuf, B * Hp, L.d_bytes, rx, rb, kSum, rank, N, lane);
    for (int r = 0; r < rounds; ++r) sent[CFB_STAGE_DOWN_PROJ] += (unsigned long long)B * p.H * tb;
    if (lane == 0 && p.traffic)
      for (int k = 0; k < CFB_STAGE_COUNT; ++k)
        if (sent[k]) atomicAdd(&p.traffic[k], sent[k]);
  }
  consumer_sync();

  // 7. O-projection over this rank's output columns into the fixed-point sum
  const int c_base = (int)rank * cols;
  consume_phase(P4, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    rowlane_item<T, QB>(it, slot, dbuf, Hp, B, lane, [&](int row, const float (&s)[QB]) {
#pragma unroll
      for (int b = 0; b < QB; ++b)
        if (b < B) red_add_fixed(&p.accum[(size_t)b * D + c_base + row], s[b]);
    });
  });
  cluster_arrive();
  cluster_wait();
}

// ---------------------------------------------------------------- host side

template <typename T, int EPL, int QB>
static int launch_mla_inst(const MlaParams& p, size_t smem, cudaStream_t st) {
  auto kern = mla_fused_kernel<T, EPL, QB>;
  if (const int rc = configure_kernel((const void*)kern, kMaxSmem, true)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.N, p.n_heads, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  LaunchAttrs at(p.N, p.flags & CFB_PDL);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

template <typename T>
static int launch_mla_t(const MlaParams& p, size_t smem, cudaStream_t st) {
  if (p.Rp == 8) {
    if (p.B == 1) return launch_mla_inst<T, 8, 1>(p, smem, st);
    if (p.B == 2) return launch_mla_inst<T, 8, 2>(p, smem, st);
    return launch_mla_inst<T, 8, 4>(p, smem, st);
  }
  if (p.B == 1) return launch_mla_inst<T, 16, 1>(p, smem, st);
  if (p.B == 2) return launch_mla_inst<T, 16, 2>(p, smem, st);
  return launch_mla_inst<T, 16, 4>(p, smem, st);
}

static int pow2_ge(int x, int lo) {
  int v = lo;
  while (v < x) v *= 2;
  return v;
}

int mla_decode(const cfb_mla_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->dtype != CFB_F16 && a->dtype != CFB_F32)
    return set_error(CFB_ERR_ARGUMENT, "dtype must be CFB_F16 (2) or CFB_F32 (4)");
  const int N = a->cluster, tb = a->dtype;
  if (N < 1 || N > 16 || (N & (N - 1)))
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16], got %d", N);
  if (a->batch < 1 || a->batch > 4) return set_error(CFB_ERR_DIMENSION, "fused_mla batch must be in [1, 4]");
  if (a->head_dim % N || a->kv_rank % N || a->hidden % N)
    return set_error(CFB_ERR_DIMENSION, "head_dim, kv_lora_rank and hidden must be divisible by %d", N);
  if (a->head_pad < a->head_dim || a->head_pad < 8 || (a->head_pad & (a->head_pad - 1)) ||
      a->head_pad * tb > 256 * 16)
    return set_error(CFB_ERR_DIMENSION, "head_pad must be a power of two >= max(8, head_dim)");
  if (a->rank_pad < a->kv_rank || a->rank_pad < 8 || (a->rank_pad & (a->rank_pad - 1)) ||
      a->rank_pad > 512)
    return set_error(CFB_ERR_DIMENSION, "rank_pad must be a power of two in [8, 512] >= kv_lora_rank");
  if ((a->hidden * tb) % 16) return set_error(CFB_ERR_DIMENSION, "hidden rows must be 16-byte multiples");
  if (a->seq_len < 0) return set_error(CFB_ERR_DIMENSION, "seq_len must be >= 0");
  if (a->seq_len == 0 && !(a->flags & CFB_APPEND))
    return set_error(CFB_ERR_DIMENSION, "no attended positions: empty cache and no appended token");
  if ((a->flags & CFB_NORM) && (!a->resid || !a->norm_w))
    return set_error(CFB_ERR_ARGUMENT, "CFB_NORM needs resid and norm_w");
  if ((!(a->flags & CFB_NORM) && !a->x) || !a->w_q || !a->w_kv || !a->w_up || !a->w_down || !a->w_out || !a->cache || !a->accum)
    return set_error(CFB_ERR_ARGUMENT, "null input / weight / accumulator pointer");
  const int rs = a->kv_rank / N, h = a->head_dim / N;
  const int rsp = pow2_ge(rs, 16 / tb);
  int spw = tuned_spw();
  MlaLayout L = mla_layout(a->batch, a->hidden, a->head_pad, a->rank_pad, rsp, N, h, rs, tb, spw);
  while (L.total > kMaxSmem && spw > 1)
    L = mla_layout(a->batch, a->hidden, a->head_pad, a->rank_pad, rsp, N, h, rs, tb, --spw);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "fused_mla schedule needs %d B of shared memory per CTA (max %d)",
                     L.total, kMaxSmem);
  MlaParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.H = a->head_dim;
  p.Hp = a->head_pad;
  p.R = a->kv_rank;
  p.Rp = a->rank_pad;
  p.rsp = rsp;
  p.N = N;
  p.n_heads = a->n_heads;
  p.S = a->seq_len;
  p.flags = a->flags;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.inv_sqrt_r = (float)(1.0 / std::sqrt((double)a->kv_rank));
  p.x = a->x;
  p.resid = a->resid;
  p.norm_w = a->norm_w;
  p.eps = a->eps;
  p.w_q = a->w_q;
  p.w_kv = a->w_kv;
  p.w_up = a->w_up;
  p.w_down = a->w_down;
  p.w_out = a->w_out;
  p.cache = a->cache;
  p.accum = a->accum;
  p.stats = a->stats;
  p.traffic = a->traffic;
  int rc = tb == 2 ? launch_mla_t<__half>(p, L.total, st) : launch_mla_t<float>(p, L.total, st);
  if (rc || !a->out) return rc;
  return mha_finalize(a->out, nullptr, a->accum, a->batch * a->hidden, st);
}

}  // namespace cfb
