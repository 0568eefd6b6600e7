// Batch>1 projections on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// At batch 16 a decode projection y = x W^T (W: M x K fp16, x: 16 x K) is a
// real dense contraction (16 flop/byte - still HBM-bound, but 16 FMAs per
// weight would saturate the CUDA cores).  Swap-AB: the weights are the MMA's
// M = 128 operand, the 16 batch rows the N = 16 operand, so one
// tcgen05.mma.cta_group::1.kind::f16 (M128 N16 K16) consumes 4 KB of weights.
//
// Work split: the (tile-major, K-minor) sequence of 16 KB weight blocks is cut
// into contiguous equal runs, one per CTA of a persistent grid; a run's part
// inside one 128-row tile is accumulated in TMEM and flushed once, so split-K
// partials only appear at tile edges (148 SMs evenly busy whatever M/128).
// Per CTA:
//   warp 0 lane 0   producer: cp.async.bulk of 16 KB weight blocks (128 rows x
//                   64 K, pre-packed on the host in the UMMA K-major
//                   no-swizzle "core matrix" order, so a plain bulk copy lands
//                   in the canonical smem layout - no tensor map needed) and
//                   the matching 2 KB activation blocks into an S-stage ring
//   warp 1 lane 0   MMA issuer: 4 x tcgen05.mma per block into a TMEM
//                   accumulator (128 lanes x 16 fp32 columns, double-buffered
//                   across units); tcgen05.commit frees ring stages and
//                   signals the epilogue
//   warps 2..5      epilogue: tcgen05.ld 32x32b.x16 (one TMEM lane quarter
//                   per warp) -> 64-bit fixed-point red.add into y_acc[n][m]
//                   (integer adds: split-K partials sum order-independently);
//                   the last CTA to finish a tile (per-tile ticket) may apply a
//                   finishing epilogue: SwiGLU + pack for the next projection,
//                   residual add, or RoPE + per-sequence KV-cache append
//
// CFB_TC_PAIR runs the same schedule on CTA pairs (cluster 2) that share each
// activation block by TMA multicast (tc_gemm_kernel<2>).
//
// Packed layouts (fp16), "core matrix" = 8 rows x 16 bytes (8 K elements):
//   W block (tile t, kb): [s = k-step (4)][c = K half (2)][g = row group (16)][8 rows][8]
//   X block (kb):         [s (4)][c (2)][g = batch group (2)][8 rows][8]
// UMMA smem descriptors (K-major, SWIZZLE_NONE): SBO = 128 B between row
// groups, LBO = 2048 B (W) / 256 B (X) between the two K core matrices.
#include <cuda_runtime.h>

#include <climits>

#include "common.h"
#include "ptx.cuh"

namespace cfb {

constexpr int kTcN = 16;            // default batch rows = MMA N (16 or 32 per launch: nb)
constexpr int kTcNMax = 32;
constexpr int kTcM = 128;           // weight rows per tile = MMA M
constexpr int kTcKB = 64;           // K elements per block
constexpr int kTcABytes = kTcM * kTcKB * 2;   // 16 KB
constexpr int kTcBBytesMax = kTcNMax * kTcKB * 2;  // 4 KB (nb = 32); nb * 128 B per block

// packed UMMA activation block layout for nb rows: element (row n, k) of
// K-block kb at [kb][s = k-step (4)][c = K half (2)][g = n / 8 (nb / 8)][n % 8][8]
__host__ __device__ __forceinline__ size_t xpack_off(int n, int k, int nb) {
  const int kb = k / kTcKB, kk = k % kTcKB, s = kk / 16, c = (kk % 16) / 8;
  return (size_t)kb * (nb * kTcKB) + (size_t)((s * 2 + c) * (nb / 8) + n / 8) * 64 + (n % 8) * 8 + (kk % 8);
}
constexpr int kTcStages = 8;
constexpr int kTcThreads = 6 * 32;

// Epilogue modes: the last CTA contributing to a 128-row tile (a per-tile
// ticket) finishes it, so no separate elementwise launch is needed.
enum TcMode { kTcAccum = 0, kTcSwiGLU = 1, kTcResidOut = 2, kTcQKV = 3 };

// kTcQKV: the projection rows are [q heads | k heads | v heads] x 128 (one tile
// = one head); the finishing CTA rounds to fp16, applies rotate-half RoPE at
// each sequence's own position (q, k), writes q for the attention kernel and
// appends k, v to that sequence's cache.
struct TcQkv {
  __half* q;              // [16][nh*128]
  __half* k_cache;        // [16][nh][cap][128]
  __half* v_cache;
  const float* rope_cs;   // [cap][64][2]
  const int* pos;         // [nb] position of the new token per sequence (-1: inactive)
  int nh, cap;
  const int* table;       // paged caches: [16][maxp] page ids (else null)
  int maxp;
};

struct TcParams {
  const __half* w;   // packed weight blocks [M/128][K/64][16 KB]
  const __half* x;   // packed activation blocks [K/64][nb * 128 B]
  unsigned long long* y;  // kTcAccum: [nb][M] fixed point (2^-32), accumulated
  float* slots;      // finishing modes: [M/128][maxc][nb][128] fp32 per-contributor partials
  int M, K, mode, nb;  // nb: batch rows = MMA N (16 or 32)
  int maxc;          // contributor slots per tile
  int* ticket;       // [M/128] zero (re-zeroed by the finishing CTA)
  __half* act;       // kTcSwiGLU: packed activations for the next projection
  float* out;        // kTcResidOut: out[n][m] = resid[n][m] + y (out may alias resid)
  const float* resid;
  TcQkv qkv;
};

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// arrive on the barrier at the same offset in every CTA of `mask` once the MMAs complete
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// global -> the same shared offset in every CTA of `mask`, completing on each one's barrier
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// finisher: value of (batch row nn, tile rows r0 .. r0 + V - 1) = sum of the
// contributors' partial slots in contributor order (deterministic); all loads
// of one contributor in flight together, everything in registers
template <int V>
__device__ __forceinline__ void tc_tile_sum(const float* tslot, int contrib, int nb, int nn, int r0,
                                            float (&v)[V]) {
  constexpr int NV = V / 4;
#pragma unroll
  for (int e = 0; e < V; ++e) v[e] = 0.f;
  for (int k = 0; k < contrib; ++k) {
    const float4* src = reinterpret_cast<const float4*>(tslot + ((size_t)k * nb + nn) * kTcM + r0);
    float4 w[NV];
#pragma unroll
    for (int e = 0; e < NV; ++e) w[e] = __ldcg(src + e);
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      v[4 * e] += w[e].x;
      v[4 * e + 1] += w[e].y;
      v[4 * e + 2] += w[e].z;
      v[4 * e + 3] += w[e].w;
    }
  }
}

// kC = 1: one CTA per run.  kC = 2 (CTA pairs, cluster 2): a pair works on
// two row-adjacent tiles over the SAME K-block run, so each activation block
// is fetched once per pair - each CTA multicasts half of it into both CTAs'
// ring slots - and a ring stage is refilled only once both CTAs' MMAs have
// released it (multicast tcgen05.commit onto both empty barriers).
template <int kC>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const TcParams p) {
  extern __shared__ __align__(1024) char smem[];
  char* sa = smem;                                   // [S][16 KB]
  char* sb = smem + kTcStages * kTcABytes;           // [S][nb * 128 B] (room for nb = 32)
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kTcStages * kTcBBytesMax);
  const int nb = p.nb, xbytes = nb * kTcKB * 2;
  uint64_t* empty = full + kTcStages;
  uint64_t* accf = empty + kTcStages;  // [2] accumulator ready
  uint64_t* acce = accf + 2;           // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // unit of work = a CTA group (kC CTAs: a cluster) = cluster ci, rank cr
  const int G = gridDim.x / kC, i = blockIdx.x / kC, cr = blockIdx.x % kC;
  // group i owns blocks [b0, b1) of the (tile-group-major, K-minor) sequence
  // of kC x 16 KB blocks: an even split; a "segment" is its run inside one
  // tile group, accumulated in TMEM and flushed once (split-K only at tile
  // boundaries).  CTA cr of the group works on tile (group * kC + cr).
  const int KBt = p.K / kTcKB, TB = (p.M / kTcM / kC) * KBt;
  const int b0 = (int)((long long)i * TB / G), b1 = (int)((long long)(i + 1) * TB / G);
  const int nseg = b1 > b0 ? (b1 - 1) / KBt - b0 / KBt + 1 : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << kC) - 1u);

  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kC);  // every CTA of the group releases the stage
    }
    mbar_init(&accf[0], 1);
    mbar_init(&accf[1], 1);
    mbar_init(&acce[0], 4);
    mbar_init(&acce[1], 4);
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: 2 accumulators x nb columns (64 allocated: nb <= 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (kC > 1) {  // the peer's barriers are initialised before anything lands on them
    cluster_arrive();
    cluster_wait();
  }
  pdl_launch_dependents();

  auto unit_kb = [&](int u, int& t, int& kb0, int& nkb) {  // segment u of this CTA
    t = b0 / KBt + u;
    const int lo = max(b0, t * KBt), hi = min(b1, (t + 1) * KBt);
    kb0 = lo - t * KBt;
    nkb = hi - lo;
  };

  if (warp == 0) {  // ------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // blocks b0 .. b1 in order (group-major, K-minor).  Weights do not depend
      // on the previous kernel: the first ring's worth streams before
      // griddepcontrol.wait, overlapping the previous kernel's tail; only the
      // activation blocks wait for it
      auto wblk = [&](int b) {  // this CTA's weight block of group block b
        return p.w + ((size_t)((b / KBt) * kC + cr) * KBt + b % KBt) * (kTcABytes / 2);
      };
      const int xs = xbytes / kC;  // this CTA's slice of each activation block
      auto xload = [&](int s, int b) {
        if constexpr (kC == 1) {
          bulk_g2s(sb + s * kTcBBytesMax, p.x + (size_t)(b % KBt) * (xbytes / 2), xbytes, &full[s],
                   policy_evict_last());
        } else {
          bulk_g2s_mc(sb + s * kTcBBytesMax + cr * xs, p.x + (size_t)(b % KBt) * (xbytes / 2) + cr * (xs / 2), xs,
                      &full[s], kMask, policy_evict_last());
        }
      };
      const int n = b1 - b0, pre = min(n, kTcStages);
      for (int it = 0; it < pre; ++it) {
        mbar_arrive_expect_tx(&full[it], kTcABytes + xbytes);
        bulk_g2s(sa + it * kTcABytes, wblk(b0 + it), kTcABytes, &full[it], pol);
      }
      pdl_wait();
      for (int it = 0; it < pre; ++it) xload(it, b0 + it);
      for (int it = pre; it < n; ++it) {
        const int s = it % kTcStages, b = b0 + it;
        mbar_wait(&empty[s], ((it / kTcStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kTcABytes + xbytes);
        bulk_g2s(sa + s * kTcABytes, wblk(b), kTcABytes, &full[s], pol);
        xload(s, b);
      }
      if constexpr (kC > 1) {
        // drain: every peer's final release of our stages has arrived before
        // this CTA may exit (their MMAs arrive on our empty barriers)
        for (int it = max(n - kTcStages, 0); it < n; ++it) mbar_wait(&empty[it % kTcStages], (it / kTcStages) & 1);
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer
    if (lane == 0) {
      // kind::f16, D f32, A/B f16 K-major, N = nb, M = 128
      const uint32_t idesc = (1u << 4) | ((uint32_t)(nb >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
      int it = 0, n = 0;
      for (int u = 0; u < nseg; ++u, ++n) {
        int t, kb0, nkb;
        unit_kb(u, t, kb0, nkb);
        const int a = n & 1;
        if (n >= 2) mbar_wait(&acce[a], ((n >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dt = tmem + (uint32_t)(a * nb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kTcStages;
          mbar_wait(&full[s], (it / kTcStages) & 1);
          tc_fence_after();
          const uint32_t abase = smem_u32(sa + s * kTcABytes), bbase = smem_u32(sb + s * kTcBBytesMax);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // X: k-step stride nb*32 B, K halves nb*16 B apart
            tc_mma(dt, umma_desc(abase + ks * 4096, 2048, 128),
                   umma_desc(bbase + ks * (nb * 32), (uint32_t)(nb * 16), 128), idesc, (kb | ks) ? 1u : 0u);
          if constexpr (kC == 1)
            tc_commit(&empty[s]);  // stage free once these MMAs have read it
          else
            tc_commit_mc(&empty[s], kMask);  // ... in both CTAs of the pair (each refills half of X)
        }
        tc_commit(&accf[a]);      // accumulator complete
      }
    }
  } else {  // -------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int n = 0;
    for (int u = 0; u < nseg; ++u, ++n) {
      int g, kb0, nkb;
      unit_kb(u, g, kb0, nkb);
      const int t = g * kC + cr;  // this CTA's tile of group g
      const int a = n & 1;
      mbar_wait(&accf[a], (n >> 1) & 1);
      tc_fence_after();
      const int m = t * kTcM + 32 * q + lane;
      uint32_t r[kTcNMax];  // this lane's row m, batch rows 0..nb-1 (16 columns per tcgen05.ld)
#pragma unroll
      for (int h16 = 0; h16 < kTcNMax / 16; ++h16)
        if (16 * h16 < nb)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(r[16 * h16 + 0]), "=r"(r[16 * h16 + 1]), "=r"(r[16 * h16 + 2]), "=r"(r[16 * h16 + 3]),
                "=r"(r[16 * h16 + 4]), "=r"(r[16 * h16 + 5]), "=r"(r[16 * h16 + 6]), "=r"(r[16 * h16 + 7]),
                "=r"(r[16 * h16 + 8]), "=r"(r[16 * h16 + 9]), "=r"(r[16 * h16 + 10]), "=r"(r[16 * h16 + 11]),
                "=r"(r[16 * h16 + 12]), "=r"(r[16 * h16 + 13]), "=r"(r[16 * h16 + 14]), "=r"(r[16 * h16 + 15])
              : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * nb + 16 * h16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[a]);  // accumulator drained: the MMA warp may reuse it
      if (p.mode == kTcAccum) {
#pragma unroll
        for (int c = 0; c < kTcNMax; ++c)
          if (c < nb) red_add_fixed(p.y + (size_t)c * p.M + m, __uint_as_float(r[c]));
        continue;
      }
      // finishing modes: this contributor's partial tile -> its own slot (plain,
      // coalesced stores: lanes = consecutive rows), summed by the finisher in
      // contributor order - deterministic, and no atomics on the critical tail
      // contributors of tile t = the groups whose runs cross tile group g
      auto cta_of = [&](long long b) { return (int)(((b + 1) * G - 1) / TB); };
      const int first = cta_of((long long)g * KBt);
      float* myslot = p.slots + ((size_t)t * p.maxc + (i - first)) * (size_t)(nb * kTcM);
#pragma unroll
      for (int c = 0; c < kTcNMax; ++c)
        if (c < nb) myslot[c * kTcM + 32 * q + lane] = __uint_as_float(r[c]);
      // ticket: the last contributor to tile t finishes it
      __threadfence();
      named_bar_sync(2, 128);
      int* flag = reinterpret_cast<int*>(tmem_slot + 1);
      const int contrib = cta_of((long long)(g + 1) * KBt - 1) - first + 1;
      if (warp == 2 && lane == 0) {
        const int old = atomicAdd(p.ticket + t, 1);
        *flag = old == contrib - 1;
        if (old == contrib - 1) p.ticket[t] = 0;
      }
      named_bar_sync(2, 128);
      if (!*flag) continue;
      __threadfence();
      // tile value (batch row nn, tile row r0 .. r0 + 4*NV - 1): sum of the
      // contributors' slots in order; all loads of a contributor in flight together
      const float* tslot = p.slots + (size_t)t * p.maxc * (nb * kTcM);
      auto tile_vals = [&](int nn, int r0, auto& v) { tc_tile_sum(tslot, contrib, nb, nn, r0, v); };
      const int et = tid - 64;  // 0..127: 16 batch rows per pass
      for (int hb = 0; hb < nb; hb += 16) {
      if (p.mode == kTcQKV) {
        // thread = (sequence nn, 8 rotation pairs (i, i + 64), i in [i0, i0 + 8))
        const int nn = hb + (et >> 3), i0 = (et & 7) * 8;
        const TcQkv& Q = p.qkv;
        const int kind = t / Q.nh, hd = t % Q.nh, ps_ = Q.pos[nn];
        const int ps = ps_ < 0 ? 0 : ps_;  // inactive sequence (position -1): no RoPE row, no cache write
        // the rotation pairs of rows i0..i0+7 are issued before the slot sums,
        // so their round trip overlaps the partial loads
        float4 cs4[4];
        if (kind < 2) {
          const float4* src = reinterpret_cast<const float4*>(Q.rope_cs + ((size_t)ps * 64 + i0) * 2);
#pragma unroll
          for (int e = 0; e < 4; ++e) cs4[e] = __ldg(src + e);
        }
        const float* csf = reinterpret_cast<const float*>(cs4);
        float lo[8], hi[8];
        tile_vals(nn, i0, lo);
        tile_vals(nn, 64 + i0, hi);
        __align__(16) __half a[8], b[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float x1 = round_to<__half>(lo[e]);
          float x2 = round_to<__half>(hi[e]);
          if (kind < 2) {  // q, k: rotate-half RoPE at the sequence's position
            const float c = csf[2 * e], sn = csf[2 * e + 1];
            const float r1 = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, sn));
            const float r2 = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, sn));
            x1 = r1;
            x2 = r2;
          }
          a[e] = __float2half_rn(x1);
          b[e] = __float2half_rn(x2);
        }
        __half* dst = nullptr;
        if (kind == 0) {
          dst = Q.q + (size_t)nn * Q.nh * 128 + hd * 128;
        } else if (ps_ >= 0) {
          // never write outside the sequence's cache: an unassigned page (-1) or a
          // position past the capacity drops the row (the host rejects both)
          __half* cache = kind == 1 ? Q.k_cache : Q.v_cache;
          if (Q.table) {
            const int pg = ps / 128 < Q.maxp ? Q.table[nn * Q.maxp + ps / 128] : -1;
            if (pg >= 0) dst = cache + (((size_t)pg * Q.nh + hd) * 128 + ps % 128) * 128;
          } else if (ps < Q.cap) {
            dst = cache + (((size_t)nn * Q.nh + hd) * Q.cap + ps) * 128;
          }
        }
        if (dst) {
          *reinterpret_cast<uint4*>(dst + i0) = *reinterpret_cast<const uint4*>(a);
          *reinterpret_cast<uint4*>(dst + 64 + i0) = *reinterpret_cast<const uint4*>(b);
        }
      } else if (p.mode == kTcSwiGLU) {
        // tile rows: 64 gate rows (f = 64t + j) then the 64 matching up rows;
        // f-range of tile t = K-block t of the next projection.  All loads of a
        // thread are issued before any store (no serialised L2 round trips).
        const int nn = hb + (et >> 3), j0 = (et & 7) * 8;  // 16 rows x 8 chunks = 128 threads
        float gv[8], uv[8];
        tile_vals(nn, j0, gv);
        tile_vals(nn, 64 + j0, uv);
        __align__(16) __half h[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          h[e] = __float2half_rn(__fmul_rn(__fdiv_rn(gv[e], __fadd_rn(1.0f, expf(-gv[e]))), uv[e]));
        *reinterpret_cast<uint4*>(p.act + xpack_off(nn, t * kTcKB + j0, nb)) = *reinterpret_cast<const uint4*>(h);
      } else {
        // 16 rows x 128 columns: thread = (row, 16-column run)
        const int nn = hb + (et >> 3), c0 = (et & 7) * 16;
        const size_t o = (size_t)nn * p.M + t * kTcM + c0;
        float4 rv[4];  // the residual does not depend on the slots: its loads go first
#pragma unroll
        for (int e = 0; e < 4; ++e)
          rv[e] = p.resid ? __ldcg(reinterpret_cast<const float4*>(p.resid + o) + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        float yv[16];
        tile_vals(nn, c0, yv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 r4 = rv[e];
          reinterpret_cast<float4*>(p.out + o)[e] =
              make_float4(__fadd_rn(r4.x, yv[4 * e]), __fadd_rn(r4.y, yv[4 * e + 1]),
                          __fadd_rn(r4.z, yv[4 * e + 2]), __fadd_rn(r4.w, yv[4 * e + 3]));
        }
      }
      }  // row passes
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kC > 1) {  // no CTA leaves while its peer may still multicast into it
    cluster_arrive();
    cluster_wait();
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
  }
}

// x [nb][K] fp16 row-major -> packed UMMA blocks (see header).
__global__ void tc_pack_x_kernel(const __half* x, __half* xp, int K, int nb) {
  pdl_wait();
  pdl_launch_dependents();
  const int nvec = nb * K / 8;  // 16-byte vectors
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x) {
    const int n = v / (K / 8), k = (v % (K / 8)) * 8;  // row n, elements k..k+7
    *reinterpret_cast<uint4*>(xp + xpack_off(n, k, nb)) = *reinterpret_cast<const uint4*>(x + (size_t)n * K + k);
  }
}

// y_acc fixed point [16][M] -> out fp32 [16][M] (optionally + resid), re-zeroes y_acc
__global__ void tc_finish_kernel(unsigned long long* yacc, float* out, const float* resid, int n) {
  pdl_wait();
  pdl_launch_dependents();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float v = fixed_to_float(yacc[i]);
    yacc[i] = 0ull;
    out[i] = resid ? __fadd_rn(resid[i], v) : v;
  }
}

int tc_smem_bytes() { return kTcStages * (kTcABytes + kTcBBytesMax) + (4 * kTcStages + 8) * 8 + 32; }

// contributor slots per tile of the even split of G CTAs in groups of kC:
// <= ceil(groups / tile groups) + 1
static int tc_maxc(int M, int K, int G, int kC = 1) {
  const int tiles = M / kTcM / kC, TB = tiles * (K / kTcKB);
  G /= kC;
  if (G > TB) G = TB;
  return (G + tiles - 1) / tiles + 1;
}
static int tc_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return sms;
}
// floats of the finishing modes' partial-slot workspace for one projection
size_t tc_slots_floats(int M, int K, int nb) {
  if (M < kTcM || K < kTcKB) return 0;
  int mc = tc_maxc(M, K, tc_sms());
  if ((M / kTcM) % 2 == 0 && tc_maxc(M, K, tc_sms(), 2) > mc) mc = tc_maxc(M, K, tc_sms(), 2);  // CTA pairs
  return (size_t)(M / kTcM) * mc * nb * kTcM;
}

int tc_gemm(const __half* w, const __half* xpacked, unsigned long long* y, int M, int K, int grid,
            cudaStream_t st, bool pdl, int mode = kTcAccum, int* ticket = nullptr, __half* act = nullptr,
            float* out = nullptr, const float* resid = nullptr, const TcQkv* qkv = nullptr, int nb = kTcN,
            float* slots = nullptr, int pair = 0) {
  if (nb != 16 && nb != 32) return set_error(CFB_ERR_DIMENSION, "tcgen05 batch must be 16 or 32");
  if (mode != kTcAccum && !slots) return set_error(CFB_ERR_ARGUMENT, "tc_gemm: finishing modes need the slot workspace");
  if (mode != kTcAccum && !ticket) return set_error(CFB_ERR_ARGUMENT, "tc_gemm: finishing modes need a ticket array");
  if (M % kTcM || K % kTcKB) return set_error(CFB_ERR_DIMENSION, "tc_gemm: M %% 128 and K %% 64 must be 0");
  // CTA pairs need an even tile count (a pair = two row-adjacent tiles)
  const int kC = (pair && (M / kTcM) % 2 == 0) ? 2 : 1;
  auto kern = kC == 2 ? tc_gemm_kernel<2> : tc_gemm_kernel<1>;
  if (const int rc = configure_kernel((const void*)kern, tc_smem_bytes(), false)) return rc;
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (grid <= 0 || grid > sms) grid = sms;
  grid = grid / kC * kC;
  const int TB = (M / kTcM) * (K / kTcKB);  // blocks; a pair takes two at a time
  TcParams p;
  p.w = w;
  p.x = xpacked;
  p.y = y;
  p.M = M;
  p.K = K;
  p.mode = mode;
  p.nb = nb;
  p.slots = slots;
  p.maxc = tc_maxc(M, K, grid, kC);
  p.ticket = ticket;
  p.act = act;
  p.out = out;
  p.resid = resid;
  p.qkv = qkv ? *qkv : TcQkv{};
  if (mode == kTcQKV && (!qkv || M != 3 * qkv->nh * kTcM))
    return set_error(CFB_ERR_DIMENSION, "tc_gemm QKV mode: M must be 3 * n_heads * 128");
  if (grid > TB) grid = TB;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kTcThreads, 1, 1);
  cfg.dynamicSmemBytes = tc_smem_bytes();
  cfg.stream = st;
  LaunchAttrs at(kC > 1 ? kC : 0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

int tc_pack_x(const __half* x, __half* xp, int K, cudaStream_t st, bool pdl, int nb = kTcN) {
  if (K % kTcKB) return set_error(CFB_ERR_DIMENSION, "tc_pack_x: K %% 64 must be 0");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((nb * K / 8 + 255) / 256, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, tc_pack_x_kernel, x, xp, K, nb));
  return CFB_OK;
}

int tc_finish(unsigned long long* yacc, float* out, const float* resid, int n, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + 255) / 256, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, tc_finish_kernel, yacc, out, resid, n));
  return CFB_OK;
}

// ---------------------------------------------------------------- batch-16 FFN
// x = f16(rmsnorm(resid[n]) * g) written straight into the packed UMMA layout
// (one CTA per batch row).
__global__ void tc_rmsnorm_pack_kernel(const float* resid, const __half* g, __half* xp, int D, float eps, int nb) {
  pdl_wait();
  pdl_launch_dependents();
  // one CTA per batch row; thread = 16 consecutive elements, loaded once
  // (4 x 16 B of the residual, 2 x 16 B of the gain) before any arithmetic
  const int n = blockIdx.x, tid = threadIdx.x;
  __shared__ float red[32];
  const float* r = resid + (size_t)n * D;
  const int k0 = tid * 16;
  const bool act = k0 < D;
  float4 rv[4];
  uint4 gv[2];
#pragma unroll
  for (int e = 0; e < 4; ++e) rv[e] = act ? __ldcg(reinterpret_cast<const float4*>(r + k0) + e) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int e = 0; e < 2; ++e) gv[e] = act ? __ldg(reinterpret_cast<const uint4*>(g + k0) + e) : make_uint4(0, 0, 0, 0);
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    ss = fmaf(rv[e].w, rv[e].w, fmaf(rv[e].z, rv[e].z, fmaf(rv[e].y, rv[e].y, fmaf(rv[e].x, rv[e].x, ss))));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  if (!act) return;
  const float inv = 1.0f / sqrtf(__fdiv_rn(tot, (float)D) + eps);
  const float* rf = reinterpret_cast<const float*>(rv);
  const __half* gh = reinterpret_cast<const __half*>(gv);
#pragma unroll
  for (int half8 = 0; half8 < 2; ++half8) {
    __align__(16) __half h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      h[e] = __float2half_rn(__fmul_rn(__fmul_rn(rf[half8 * 8 + e], inv), __half2float(gh[half8 * 8 + e])));
    *reinterpret_cast<uint4*>(xp + xpack_off(n, k0 + half8 * 8, nb)) = *reinterpret_cast<const uint4*>(h);
  }
}

__global__ void tc_advance_kernel(int* pos, int nb) {  // every active sequence moves to its next position
  pdl_wait();
  if ((int)threadIdx.x < nb && pos[threadIdx.x] >= 0) pos[threadIdx.x] += 1;
}

template <class K, class... Args>
static int launch_simple(K kern, dim3 grid, int block, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block, 1, 1);
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
  return CFB_OK;
}

int ffn_b16(const cfb_ffn_b16_args* a, cudaStream_t st) {
  if (!a || !a->resid || !a->norm_w || !a->w_gu || !a->w_dn || !a->xp || !a->gu_acc || !a->ap ||
      !a->out_acc || !a->slots)
    return set_error(CFB_ERR_ARGUMENT, "null pointer");
  const int D = a->hidden, F = a->inter;
  if (D % 128 || F % 64 || (2 * F) % 128)
    return set_error(CFB_ERR_DIMENSION, "ffn_b16: hidden %% 128 and inter %% 64 must be 0");
  if (!a->ticket) return set_error(CFB_ERR_ARGUMENT, "ffn_b16: null ticket workspace");
  const int nb = a->batch ? a->batch : kTcN;
  if (nb != 16 && nb != 32) return set_error(CFB_ERR_DIMENSION, "ffn_b16: batch must be 16 or 32");
  const bool pdl = a->flags & CFB_PDL;
  int rc;
  if ((rc = launch_simple(tc_rmsnorm_pack_kernel, nb, (D / 16 + 31) / 32 * 32, st, pdl, a->resid,
                          static_cast<const __half*>(a->norm_w), static_cast<__half*>(a->xp), D, a->eps, nb)))
    return rc;
  // gate/up tiles interleave 64 gate + 64 up rows, finished (SwiGLU + pack) by
  // their last contributor; down tiles finished as resid + sum
  const int pair = (a->flags & CFB_TC_PAIR) ? 1 : 0;
  if ((rc = tc_gemm(static_cast<const __half*>(a->w_gu), static_cast<const __half*>(a->xp), a->gu_acc,
                    2 * F, D, 0, st, true, kTcSwiGLU, a->ticket, static_cast<__half*>(a->ap), nullptr, nullptr,
                    nullptr, nb, a->slots, pair)))
    return rc;
  return tc_gemm(static_cast<const __half*>(a->w_dn), static_cast<const __half*>(a->ap), a->out_acc, D, F,
                 0, st, true, kTcResidOut, a->ticket + 2 * F / kTcM, nullptr, a->resid,
                 (a->flags & CFB_PARTIAL) ? nullptr : a->resid, nullptr, nb, a->slots, pair);
}

int batch_attention(const __half* q, const __half* kc, const __half* vc, const int* pos, int nh, int cap,
                    int max_len, float* part, int* ticket, __half* xp, const int* table, int maxp,
                    cudaStream_t st, bool pdl, int nb);

// One Llama decoder layer for 16 independent sequences (7 PDL-chained launches):
// RMSNorm+pack -> QKV projection (RoPE + per-sequence cache append in the
// finishing epilogue) -> split-KV attention + merge (packed) -> O projection
// (+ residual) -> batch-16 FFN block.
int llama_b16_layer(const cfb_b16_layer_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  const int D = a->hidden, nh = a->n_heads, F = a->inter, Ka = nh * 128;
  if (Ka > D || D % 128 || F % 64 || a->stage < 0 || a->stage > 2)
    return set_error(CFB_ERR_DIMENSION, "b16 layer: n_heads*128 <= hidden, hidden %% 128, inter %% 64");
  const bool pdl = a->flags & CFB_PDL, partial = a->flags & CFB_PARTIAL;
  const int pair = (a->flags & CFB_TC_PAIR) ? 1 : 0;
  const int nb = a->batch ? a->batch : kTcN;
  if (nb != 16 && nb != 32) return set_error(CFB_ERR_DIMENSION, "batched layer: batch must be 16 or 32");
  const int Mq = 3 * nh * 128;
  int rc;
  if (a->stage != 2) {  // attention half
    if ((rc = launch_simple(tc_rmsnorm_pack_kernel, nb, (D / 16 + 31) / 32 * 32, st, pdl, (const float*)a->resid,
                            static_cast<const __half*>(a->attn_norm), static_cast<__half*>(a->xp), D, a->eps, nb)))
      return rc;
    TcQkv qkv;
    qkv.q = static_cast<__half*>(a->q16);
    qkv.k_cache = static_cast<__half*>(a->k_cache);
    qkv.v_cache = static_cast<__half*>(a->v_cache);
    qkv.rope_cs = a->rope_cs;
    qkv.pos = a->pos;
    qkv.nh = nh;
    qkv.cap = a->cache_cap;
    qkv.table = a->block_table;
    qkv.maxp = a->max_pages;
    if (a->block_table && a->max_pages * 128 < a->max_len)
      return set_error(CFB_ERR_DIMENSION, "b16 layer: max_pages * 128 < max_len");
    if ((rc = tc_gemm(static_cast<const __half*>(a->w_qkv), static_cast<const __half*>(a->xp), a->qkv_acc, Mq, D,
                      0, st, true, kTcQKV, a->ticket, nullptr, nullptr, nullptr, &qkv, nb, a->slots, pair)))
      return rc;
    if ((rc = batch_attention(static_cast<const __half*>(a->q16), static_cast<const __half*>(a->k_cache),
                              static_cast<const __half*>(a->v_cache), a->pos, nh, a->cache_cap, a->max_len,
                              a->part, a->ticket + (Mq + 2 * D + 2 * F) / kTcM, static_cast<__half*>(a->xp),
                              a->block_table, a->max_pages, st, true, nb)))
      return rc;
    if ((rc = tc_gemm(static_cast<const __half*>(a->w_o), static_cast<const __half*>(a->xp), a->o_acc, D, Ka, 0,
                      st, true, kTcResidOut, a->ticket + Mq / kTcM, nullptr, a->resid, partial ? nullptr : a->resid,
                      nullptr, nb, a->slots, pair)))
      return rc;
  }
  if (a->stage == 1) return CFB_OK;
  cfb_ffn_b16_args f = {};
  f.hidden = D;
  f.inter = F;
  f.flags = CFB_PDL | (partial ? CFB_PARTIAL : 0) | (a->flags & CFB_TC_PAIR);
  f.eps = a->eps;
  f.resid = a->resid;
  f.norm_w = a->ffn_norm;
  f.w_gu = a->w_gu;
  f.w_dn = a->w_dn;
  f.xp = a->xp;
  f.gu_acc = a->gu_acc;
  f.ap = a->ap;
  f.out_acc = a->o_acc;
  f.ticket = a->ticket + (Mq + D) / kTcM;
  f.batch = nb;
  f.slots = a->slots;
  return ffn_b16(&f, st);
}

// greedy argmax per sequence over the fixed-point logits [16][V] (fixed point
// is monotonic in the value: int64 compare; first index of the max, numpy
// semantics).  Grid (kArgSplit, 16): each CTA scans a V slice (re-zeroing the
// accumulator, optionally exporting fp32 logits) and publishes its (max, index);
// the last CTA of a sequence (ticket) reduces the partials.
constexpr int kArgSplit = 32;
__device__ __forceinline__ void arg_better(long long& bv, int& bi, long long ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
}
__device__ __forceinline__ void arg_block_reduce(long long& best, int& besti, long long* bv, int* bi) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    arg_better(best, besti, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, besti, o));
  if ((tid & 31) == 0) {
    bv[tid >> 5] = best;
    bi[tid >> 5] = besti;
  }
  __syncthreads();
  if (tid == 0)
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) arg_better(best, besti, bv[w], bi[w]);
}
__global__ void __launch_bounds__(256) tc_argmax_kernel(unsigned long long* yacc, int V, int* tokens,
                                                        float* logits, unsigned long long* scratch) {
  pdl_wait();
  pdl_launch_dependents();
  const int c = blockIdx.x, n = blockIdx.y, tid = threadIdx.x;
  __shared__ long long bv[8];
  __shared__ int bi[8];
  __shared__ int last;
  const int per = (V / 2 + kArgSplit - 1) / kArgSplit * 2, v0 = c * per, v1 = min(V, v0 + per);
  unsigned long long* row = yacc + (size_t)n * V;
  long long best = LLONG_MIN;
  int besti = 0x7fffffff;
  for (int v = v0 + 2 * tid; v < v1; v += 512) {  // V even: 16 B per thread
    const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(row + v));
    *reinterpret_cast<ulonglong2*>(row + v) = make_ulonglong2(0ull, 0ull);
    if (logits)
      *reinterpret_cast<float2*>(logits + (size_t)n * V + v) = make_float2(fixed_to_float(x.x), fixed_to_float(x.y));
    arg_better(best, besti, (long long)x.x, v);
    arg_better(best, besti, (long long)x.y, v + 1);
  }
  arg_block_reduce(best, besti, bv, bi);
  // scratch: [32][kArgSplit] values, [32][kArgSplit] indices, [32] tickets (up to 32 rows)
  unsigned long long* sv = scratch + (size_t)n * kArgSplit;
  unsigned long long* si = scratch + kTcNMax * kArgSplit + (size_t)n * kArgSplit;
  unsigned long long* tk = scratch + 2 * kTcNMax * kArgSplit + n;
  if (tid == 0) {
    sv[c] = (unsigned long long)best;
    si[c] = (unsigned long long)besti;
    __threadfence();
    const unsigned long long old = atomicAdd(tk, 1ull);
    last = old == kArgSplit - 1;
    if (last) *tk = 0ull;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  best = LLONG_MIN;
  besti = 0x7fffffff;
  if (tid < kArgSplit) {
    best = (long long)__ldcg(sv + tid);
    besti = (int)__ldcg(si + tid);
  }
  arg_block_reduce(best, besti, bv, bi);
  if (tid == 0) tokens[n] = besti;
}

int b16_lm_head(const float* resid, const __half* g, const __half* w, int V, int D, float eps, __half* xp,
                unsigned long long* yacc, int* tokens, float* logits, unsigned long long* scratch, int nb,
                cudaStream_t st) {
  if (V % kTcM || D % 128) return set_error(CFB_ERR_DIMENSION, "b16 LM head: vocab %% 128, hidden %% 128");
  if (nb != 16 && nb != 32) return set_error(CFB_ERR_DIMENSION, "batched LM head: batch must be 16 or 32");
  int rc;
  if ((rc = launch_simple(tc_rmsnorm_pack_kernel, nb, (D / 16 + 31) / 32 * 32, st, true, resid, g, xp, D, eps, nb)))
    return rc;
  if ((rc = tc_gemm(w, xp, yacc, V, D, 0, st, true, kTcAccum, nullptr, nullptr, nullptr, nullptr, nullptr, nb)))
    return rc;
  return launch_simple(tc_argmax_kernel, dim3(kArgSplit, nb), 256, st, true, yacc, V, tokens, logits, scratch);
}

}  // namespace cfb

extern "C" {

int cfb_b16_lm_head(const float* resid, const void* norm_w, const void* w_lm, int vocab, int hidden,
                    float eps, void* xp, unsigned long long* y_acc, int* tokens, float* logits,
                    unsigned long long* scratch, int batch, void* stream) {
  return cfb::b16_lm_head(resid, static_cast<const __half*>(norm_w), static_cast<const __half*>(w_lm), vocab,
                          hidden, eps, static_cast<__half*>(xp), y_acc, tokens, logits, scratch,
                          batch ? batch : cfb::kTcN, static_cast<cudaStream_t>(stream));
}

int cfb_llama_b16_layer(const cfb_b16_layer_args* args, void* stream) {
  return cfb::llama_b16_layer(args, static_cast<cudaStream_t>(stream));
}

int cfb_b16_advance(int* pos, int batch, void* stream) {
  return cfb::launch_simple(cfb::tc_advance_kernel, 1, 32, static_cast<cudaStream_t>(stream), true, pos,
                            batch ? batch : cfb::kTcN);
}


int cfb_tc_gemm_b16(const void* w_packed, const void* x, void* x_packed, unsigned long long* y_acc,
                    float* y, const float* resid, int M, int K, int flags, void* stream) {
  using namespace cfb;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!w_packed || !x || !x_packed || !y_acc) return set_error(CFB_ERR_ARGUMENT, "null pointer");
  const bool pdl = flags & CFB_PDL;
  int rc = tc_pack_x(static_cast<const __half*>(x), static_cast<__half*>(x_packed), K, st, pdl);
  if (rc) return rc;
  if ((rc = tc_gemm(static_cast<const __half*>(w_packed), static_cast<const __half*>(x_packed), y_acc,
                    M, K, 0, st, true, kTcAccum, nullptr, nullptr, nullptr, nullptr, nullptr, kTcN, nullptr,
                    (flags & CFB_TC_PAIR) ? 1 : 0)))
    return rc;
  if (!y) return CFB_OK;
  return tc_finish(y_acc, y, resid, 16 * M, st, true);
}

size_t cfb_b16_slots_floats(int hidden, int n_heads, int inter, int batch) {
  using namespace cfb;
  const int nb = batch ? batch : kTcN, Ka = n_heads * 128;
  size_t m = tc_slots_floats(3 * Ka, hidden, nb);
  const size_t c[3] = {tc_slots_floats(hidden, Ka, nb), tc_slots_floats(2 * inter, hidden, nb),
                       tc_slots_floats(hidden, inter, nb)};
  for (size_t v : c) m = v > m ? v : m;
  return m;
}

int cfb_ffn_b16(const cfb_ffn_b16_args* args, void* stream) {
  return cfb::ffn_b16(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
