// Head-batched MLA decode for the DeepSeek block engine (B = 1, 16 heads).
//
// Same math as the fused_mla dataflow (reference dataflows.py:316-429 /
// oracle.py:55-93, absorbed form, scale 1/sqrt(kv_lora_rank), the new
// token's latent row attended once) but laid out for a whole B200 instead of
// one cluster per head.  The reference dataflow re-reads W_kv (2 MB) and the
// entire latent cache once per head (dataflows.py:352-368, :393-397); here
// every weight and every cache row crosses HBM once:
//
//   mla_proj_kernel  (persistent grid)  x = f16(rmsnorm(resid) * g);
//                    [q | c] = x [W_q | W_kv]  (row-tiled GEMV, 2560 rows of D)
//                    -- grid barrier --
//                    q_lat[h] = f16(q[h] W_up[h])  (row-per-lane GEMV, 8192 rows of H)
//   mla_attn_kernel  split-KV over the S+1 latent rows: every CTA streams a
//                    contiguous chunk of rows ONCE for all 16 heads with
//                    warp-level tensor-core MMAs (mma.sync m16n8k16, heads =
//                    the M=16 dimension): S = Q_lat L^T, online softmax,
//                    Z += P L; partial (m, l, Z) per CTA
//   mla_out_kernel   (persistent grid)  merge the partials -> this CTA's z
//                    elements (fp16), and straight away their split-K share
//                    of o[h] = z[h] W_down[h] (W_down rows of those elements)
//                    into a 64-bit fixed-point o accumulator;
//                    -- grid barrier --  o = f16(o_acc); out = sum_h o[h] W_out[h]
//                    -> the fixed-point head-sum accumulator the MoE reads.
#include <cuda_runtime.h>

#include <utility>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

constexpr int kMlaHeads = 16;          // the M = 16 MMA dimension
constexpr int kAttnRows = 32;          // cache rows per attention tile
constexpr int kAttnStages = 3;
constexpr int kAttnWarps = 4;          // each owns 128 of the 512 latent dims
constexpr int kRowStride = 1040;       // 1024 B row + 16 B pad: conflict-free ldmatrix

struct MlaEngParams {
  int D, H, R, S, flags, spw, sleep_max, G2;
  int NH;                 // real heads (<= 16; tensor-parallel shard): MMA rows >= NH are zero
  float eps, scale_log2;  // scale_log2 = log2(e) / sqrt(R)
  const float* resid;
  const __half* norm_w;
  const __half* w_a;     // row tiles of [W_q^T (nh*H rows) ; W_kv^T (R rows)] x D
  const __half* w_up;    // rows h*R + j = W_up[h][:, j] (H), chunk-rotated by row
  const __half* w_dn;    // W_down [nh][R][H]: row h*R + j = W_down[h][j, :]
  const __half* w_o;     // row tiles of W_out^T: rows d = [W_out[h][:, d]]_h (nh*H)
  const __half* cache;   // [S][R]
  __half* qc;            // [nh*H + R]  q | new latent row
  __half* qlat;          // [nh][R]
  float* part;           // [G2][2*nh + nh*R]  m, l, Z per attention CTA
  unsigned long long* o_acc;  // [nh*H] fixed-point o (zeroed by the attention launch)
  unsigned long long* accum;   // [D] fixed-point head sum (plain stores)
  unsigned long long* barrier; // [2] proj, out grid barriers (monotonic)
  unsigned long long* trace;   // [grid][16] %globaltimer stamps (profiling) or null
};

// profiling stamp k of this CTA (thread 0): proj 0-4, attention 5-7, out 8-13
__device__ __forceinline__ void mla_stamp(const MlaEngParams& p, int k, int tid) {
  if (p.trace && tid == 0) p.trace[(size_t)blockIdx.x * 16 + k] = globaltimer();
}

// ------------------------------------------------------------------ kernel 1
struct MlaProjLayout {
  int bars, xs, part, qs, red, total;
};
__host__ __device__ inline MlaProjLayout mla_proj_layout(int D, int H, int G, int spw) {
  MlaProjLayout L;
  const int ta = (kMlaHeads * H + 512 + 3) / 4;  // R <= 512
  const int rows = 4 * ((ta + G - 1) / G);
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.xs = o;    o += ((D * 2 + 15) & ~15);
  L.part = o;  o += kNumConsumerWarps * rows * 4;
  L.qs = o;    o += ((kMlaHeads * H * 2 + 15) & ~15);
  L.red = o;   o += kNumConsumerWarps * 4 * 2;
  L.total = o;
  return L;
}

// Grid barrier whose counter advances by exactly kProjUnit per launch whatever
// the grid (CTA 0 arrives with the remainder): the projection's grid shrinks
// at short contexts (host side), and consecutive launches on one workspace
// may use different grids.
constexpr unsigned long long kProjUnit = 1ull << 12;
__device__ __forceinline__ void proj_barrier(unsigned long long* counter, int tid) {
  consumer_sync();
  if (tid == 0) {
    __threadfence();
    const unsigned long long inc = blockIdx.x == 0 ? kProjUnit - (gridDim.x - 1) : 1ull;
    const unsigned long long old = atomicAdd(counter, inc);
    spin_until_geq(counter, (old / kProjUnit + 1) * kProjUnit);
  }
  consumer_sync();
}

__global__ void __launch_bounds__(kThreads, 1) mla_proj_kernel(const MlaEngParams p) {
  extern __shared__ __align__(128) char smem[];
  const int D = p.D, H = p.H, R = p.R, G = gridDim.x, i = blockIdx.x;
  const MlaProjLayout L = mla_proj_layout(D, H, G, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NH = p.NH, TA = (NH * H + R) / 4;
  const int a0 = (int)((long long)i * TA / G), a1 = (int)((long long)(i + 1) * TA / G);
  // W_up rows in 32-row units (keeps each CTA's rows aligned to the chunk rotation)
  const int UB = NH * R / 32;
  const int b0 = 32 * (int)((long long)i * UB / G), b1 = 32 * (int)((long long)(i + 1) * UB / G);
  const int hb0 = b0 / R, hb1 = b1 > b0 ? (b1 - 1) / R : hb0;  // heads touched (<= 2 segments)
  auto seg = [&](int s, int& r0, int& r1) {
    const int h = hb0 + s;
    r0 = max(b0, h * R);
    r1 = min(b1, (h + 1) * R);
    return h;
  };
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const Phase PA = make_phase(p.w_a + (size_t)a0 * 4 * D, nullptr, a1 - a0, 4 * D * 2, true);
  int r0, r1;
  const int nseg = b1 > b0 ? hb1 - hb0 + 1 : 0;
  seg(0, r0, r1);
  const Phase PB0 = make_phase(p.w_up + (size_t)r0 * H, nullptr, nseg > 0 ? r1 - r0 : 0, H * 2);
  seg(1, r0, r1);
  const Phase PB1 = make_phase(p.w_up + (size_t)r0 * H, nullptr, nseg > 1 ? r1 - r0 : 0, H * 2);
  pdl_launch_dependents();
  if (warp == kNumConsumerWarps) {
    const Phase ph[3] = {PA, PB0, PB1};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  pdl_wait();
  mla_stamp(p, 0, tid);
  __half* xs = reinterpret_cast<__half*>(smem + L.xs);
  float* part = reinterpret_cast<float*>(smem + L.part);
  __half* qs = reinterpret_cast<__half*>(smem + L.qs);
  float* red = reinterpret_cast<float*>(smem + L.red);
  rmsnorm_to_smem<__half, true>(xs, p.resid, p.norm_w, 1, D, p.eps, red, tid);
  mla_stamp(p, 1, tid);
  int cnt = 0;
  const int rows = 4 * (a1 - a0);
  tiled_gemv_phase<__half, 1, true>(PA, ring, warp, lane, tid, cnt, xs, D, 1, rows, part,
                                    [&](int row, int, float v) {
                                      p.qc[4 * a0 + row] = __float2half_rn(v);
                                    });
  mla_stamp(p, 2, tid);
  proj_barrier(p.barrier, tid);
  mla_stamp(p, 3, tid);
  for (int t = tid; t < NH * H / 8; t += kConsumerThreads)
    reinterpret_cast<uint4*>(qs)[t] = __ldcg(reinterpret_cast<const uint4*>(p.qc) + t);
  consumer_sync();
  for (int s = 0; s < 2; ++s) {
    const int h = seg(s, r0, r1);
    const Phase& P = s == 0 ? PB0 : PB1;
    consume_phase(P, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
      rowlane_item<__half, 1>(it, slot, qs + (size_t)h * H, H, 1, lane,
                              [&](int g, const float (&v)[1]) {
                                p.qlat[(size_t)r0 + g] = __float2half_rn(v[0]);
                              });
    });
  }
  consumer_sync();
  mla_stamp(p, 4, tid);
}

// ------------------------------------------------------------------ kernel 2
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

constexpr int kAttnThreads = kAttnWarps * 32;
constexpr int kAttnStage = kAttnRows * kRowStride;
constexpr int kAttnSmem = kAttnStages * kAttnStage + kMlaHeads * kRowStride +
                          kAttnWarps * kMlaHeads * kAttnRows * 4 + 64;

// grid G2: CTA c attends rows [c*T/G2, (c+1)*T/G2) of the T = S + 1 rows
// (cache rows, then the new latent row).  Requires R = 512, 16 heads.
__global__ void __launch_bounds__(kAttnThreads) mla_attn_kernel(const MlaEngParams p) {
  extern __shared__ __align__(128) char smem[];
  char* stages = smem;
  char* qsm = smem + kAttnStages * kAttnStage;
  float* spart = reinterpret_cast<float*>(qsm + kMlaHeads * kRowStride);
  uint64_t* full = reinterpret_cast<uint64_t*>(spart + kAttnWarps * kMlaHeads * kAttnRows);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int S = p.S, T = S + 1, c = blockIdx.x, G2 = gridDim.x;
  const int j0 = (int)((long long)c * T / G2), j1 = (int)((long long)(c + 1) * T / G2);
  const int ntiles = (j1 - j0 + kAttnRows - 1) / kAttnRows;
  // zero the stages once: rows past the chunk end stay finite (P = 0 there)
  for (int k = tid; k < kAttnStages * kAttnStage / 16; k += kAttnThreads)
    reinterpret_cast<uint4*>(stages)[k] = make_uint4(0, 0, 0, 0);
  if (tid == 0)
    for (int s = 0; s < kAttnStages; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int tile) {  // thread 0: TMA row copies of one tile
    const int s = tile % kAttnStages, r0 = j0 + tile * kAttnRows;
    const int n = min(kAttnRows, j1 - r0);
    mbar_arrive_expect_tx(&full[s], (uint32_t)(n * 1024));
    for (int r = 0; r < n; ++r) {
      const int j = r0 + r;
      const void* src = j < S ? (const void*)(p.cache + (size_t)j * 512)
                              : (const void*)(p.qc + p.NH * p.H);  // new latent row
      bulk_g2s(stages + s * kAttnStage + r * kRowStride, src, 1024, &full[s], pol);
    }
  };
  pdl_launch_dependents();
  if (tid == 0)  // cache rows do not depend on the previous kernel: stream them now
    for (int k = 0; k < min(kAttnStages - 1, ntiles); ++k)
      if (j0 + k * kAttnRows + kAttnRows <= S) issue(k);
  pdl_wait();
  mla_stamp(p, 5, tid);
  // o_acc's previous reader (the last step's mla_out) completed long before
  // this launch; its next writers (this step's mla_out) start after it
  for (int t = c * kAttnThreads + tid; t < p.NH * p.H; t += G2 * kAttnThreads) p.o_acc[t] = 0ull;
  if (tid == 0)
    for (int k = 0; k < min(kAttnStages - 1, ntiles); ++k)
      if (j0 + k * kAttnRows + kAttnRows > S) issue(k);  // tiles holding the new row
  // q_lat (NH x 512 fp16, zero rows up to 16) -> smem rows of kRowStride
  {  // all 8 loads of a thread in flight together (one L2 round trip, not 8)
    constexpr int kPer = kMlaHeads * 64 / kAttnThreads;
    uint4 v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int k = tid + j * kAttnThreads, h = k >> 6, ch = k & 63;
      v[j] = h < p.NH ? __ldcg(reinterpret_cast<const uint4*>(p.qlat + h * 512) + ch) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int k = tid + j * kAttnThreads, h = k >> 6, ch = k & 63;
      *reinterpret_cast<uint4*>(qsm + h * kRowStride + ch * 16) = v[j];
    }
  }
  __syncthreads();
  // A fragments of this warp's 128 dims (8 k-steps of 16)
  uint32_t qa[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
    ldsm_x4(qa[ks], qsm + (lane & 15) * kRowStride + (warp * 128 + ks * 16 + 8 * (lane >> 4)) * 2);
  float zacc[16][4];
#pragma unroll
  for (int nb = 0; nb < 16; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) zacc[nb][e] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // rows g, g + 8
  mla_stamp(p, 6, tid);

  for (int tile = 0; tile < ntiles; ++tile) {
    if (tid == 0 && tile + kAttnStages - 1 < ntiles) issue(tile + kAttnStages - 1);
    const int s = tile % kAttnStages;
    mbar_wait(&full[s], (tile / kAttnStages) & 1);
    const char* st = stages + s * kAttnStage;
    // partial scores over this warp's dims: 16 heads x 32 rows
    float sc[4][4];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[nb][e] = 0.f;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
#pragma unroll
      for (int ks = 0; ks < 8; ks += 2) {
        // x4: rows 8nb + (lane & 7), k offsets 0/8 of k-steps ks and ks+1
        uint32_t b[4];
        ldsm_x4(b, st + (8 * nb + (lane & 7)) * kRowStride +
                       (warp * 128 + ks * 16 + 8 * (lane >> 3)) * 2);
        mma16816(sc[nb], qa[ks], b[0], b[1]);
        mma16816(sc[nb], qa[ks + 1], b[2], b[3]);
      }
    }
    float* my = spart + warp * kMlaHeads * kAttnRows;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      my[g * kAttnRows + 8 * nb + 2 * t4] = sc[nb][0];
      my[g * kAttnRows + 8 * nb + 2 * t4 + 1] = sc[nb][1];
      my[(g + 8) * kAttnRows + 8 * nb + 2 * t4] = sc[nb][2];
      my[(g + 8) * kAttnRows + 8 * nb + 2 * t4 + 1] = sc[nb][3];
    }
    __syncthreads();
    const int nvalid = min(kAttnRows, j1 - j0 - tile * kAttnRows);
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = g + 8 * (e >> 1), col = 8 * nb + 2 * t4 + (e & 1);
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) v += spart[(w * kMlaHeads + row) * kAttnRows + col];
        sc[nb][e] = col < nvalid ? v * p.scale_log2 : -INFINITY;
      }
    // online softmax (base 2; the scale carries log2 e / sqrt(R))
    float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      mt[0] = fmaxf(mt[0], fmaxf(sc[nb][0], sc[nb][1]));
      mt[1] = fmaxf(mt[1], fmaxf(sc[nb][2], sc[nb][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mt[r] = fmaxf(mt[r], __shfl_xor_sync(0xffffffffu, mt[r], 1));
      mt[r] = fmaxf(mt[r], __shfl_xor_sync(0xffffffffu, mt[r], 2));
    }
    float alpha[2], mnew[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(m_run[r], mt[r]);
      alpha[r] = m_run[r] == -INFINITY ? 0.f : exp2f(m_run[r] - mnew[r]);
      m_run[r] = mnew[r];
    }
    float ls[2] = {0.f, 0.f};
    uint32_t pa[2][4];  // P as A fragments: k-steps of 16 rows
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      const float p0 = exp2f(sc[nb][0] - mnew[0]), p1 = exp2f(sc[nb][1] - mnew[0]);
      const float p2 = exp2f(sc[nb][2] - mnew[1]), p3 = exp2f(sc[nb][3] - mnew[1]);
      ls[0] += p0 + p1;
      ls[1] += p2 + p3;
      pa[nb >> 1][(nb & 1) * 2 + 0] = pack_h2(p0, p1);
      pa[nb >> 1][(nb & 1) * 2 + 1] = pack_h2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      ls[r] += __shfl_xor_sync(0xffffffffu, ls[r], 1);
      ls[r] += __shfl_xor_sync(0xffffffffu, ls[r], 2);
      l_run[r] = l_run[r] * alpha[r] + ls[r];
    }
#pragma unroll
    for (int nb = 0; nb < 16; ++nb) {
      zacc[nb][0] *= alpha[0];
      zacc[nb][1] *= alpha[0];
      zacc[nb][2] *= alpha[1];
      zacc[nb][3] *= alpha[1];
    }
    // Z[:, dims of this warp] += P (16 x 32) . L_tile (32 x 128)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int nb = 0; nb < 16; nb += 2) {
        // x4.trans: rows 16ks + (lane & 15), dims 8nb + 8*(lane >> 4)
        uint32_t b[4];
        ldsm_x4_t(b, st + (16 * ks + (lane & 15)) * kRowStride +
                         (warp * 128 + 8 * nb + 8 * (lane >> 4)) * 2);
        mma16816(zacc[nb], pa[ks], b[0], b[1]);
        mma16816(zacc[nb + 1], pa[ks], b[2], b[3]);
      }
    }
    __syncthreads();  // stage s and spart are reused
  }
  // partial: m, l (base-2 units) per head, unnormalised Z
  float* out = p.part + (size_t)c * (2 * kMlaHeads + kMlaHeads * 512);
  if (warp == 0 && t4 == 0) {
    out[g] = m_run[0];
    out[g + 8] = m_run[1];
    out[kMlaHeads + g] = l_run[0];
    out[kMlaHeads + g + 8] = l_run[1];
  }
  float* z = out + 2 * kMlaHeads;
#pragma unroll
  for (int nb = 0; nb < 16; ++nb) {
    const int d = warp * 128 + 8 * nb + 2 * t4;
    *reinterpret_cast<float2*>(z + g * 512 + d) = make_float2(zacc[nb][0], zacc[nb][1]);
    *reinterpret_cast<float2*>(z + (g + 8) * 512 + d) = make_float2(zacc[nb][2], zacc[nb][3]);
  }
  mla_stamp(p, 7, tid);
}

// ------------------------------------------------------------------ kernel 3
struct MlaOutLayout {
  int bars, zs, os, part, total;
};
__host__ __device__ inline MlaOutLayout mla_out_layout(int D, int H, int G, int spw) {
  MlaOutLayout L;
  const int to = (D / 4 + G - 1) / G;
  const int rows = 4 * to;
  int o = ring_bytes(spw);
  L.bars = o;  o += 2 * kNumSlots * 8;
  L.zs = o;    o += kMlaHeads * 512 * 2;
  L.os = o;    o += kMlaHeads * H * 2;
  L.part = o;  o += kNumConsumerWarps * rows * 4;
  L.total = o;
  return L;
}

__global__ void __launch_bounds__(kThreads, 1) mla_out_kernel(const MlaEngParams p) {
  extern __shared__ __align__(128) char smem[];
  const int D = p.D, H = p.H, R = p.R, G = gridDim.x, i = blockIdx.x, G2 = p.G2;
  const MlaOutLayout L = mla_out_layout(D, H, G, p.spw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NH = p.NH;
  // z elements [e0, e1) of the NH*R (head-major) merge; their W_down rows
  // are the same indices of the [NH*R][H] layout, cut at the head boundary
  const int NZ = NH * R;
  const int e0 = (int)((long long)i * NZ / G), e1 = (int)((long long)(i + 1) * NZ / G);
  const int h0 = e0 / R, h1 = (e1 - 1) / R;
  auto eseg = [&](int s, int& a, int& b) {
    const int h = h0 + s;
    a = max(e0, h * R);
    b = min(e1, (h + 1) * R);
    return h;
  };
  const int TO = D / 4;
  const int o0 = (int)((long long)i * TO / G), o1 = (int)((long long)(i + 1) * TO / G);
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  // 8 rows per item (not a full 32-row slot) so the ~56 rows spread over 7 warps
  auto rows8 = [](Phase P) {
    P.per_item = 8;
    P.n_items = (P.n_units + 7) / 8;
    return P;
  };
  int ea, eb;
  eseg(0, ea, eb);
  const Phase PD0 = rows8(make_phase(p.w_dn + (size_t)ea * H, nullptr, max(eb - ea, 0), H * 2));
  eseg(1, ea, eb);
  const Phase PD1 = rows8(make_phase(p.w_dn + (size_t)ea * H, nullptr, h1 > h0 ? max(eb - ea, 0) : 0, H * 2));
  const Phase PO = make_phase(p.w_o + (size_t)o0 * 4 * NH * H, nullptr, o1 - o0, 4 * NH * H * 2, true);
  pdl_launch_dependents();
  if (warp == kNumConsumerWarps) {
    const Phase ph[3] = {PD0, PD1, PO};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  pdl_wait();
  mla_stamp(p, 8, tid);
  __half* zs = reinterpret_cast<__half*>(smem + L.zs);
  __half* os = reinterpret_cast<__half*>(smem + L.os);
  float* part = reinterpret_cast<float*>(smem + L.part);
  // 1. merge the attention partials for this CTA's slice of z (16 x 512):
  //    per head (<= 2 per CTA) the weights w_q = 2^(m_q - M) and 1 / sum_q w_q l_q
  //    once into smem, then per element the sum over q split across a warp's
  //    lanes, 4 elements per pass so their loads are in flight together
  float* zloc = reinterpret_cast<float*>(zs) + 2048;  // [e1 - e0 <= 512] merged z (fp16 values)
  {
    const int stride = 2 * kMlaHeads + kMlaHeads * 512;
    float* wq = reinterpret_cast<float*>(zs);  // [2][G2] weights, then [2] 1/l
    if (warp < 2 && h0 + warp <= h1) {
      const int h = h0 + warp;
      float mv[5], lv[5];  // G2 <= 160: all of a lane's (m, l) loads in flight together
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int q = lane + 32 * j;
        mv[j] = q < G2 ? __ldcg(p.part + (size_t)q * stride + h) : -INFINITY;
        lv[j] = q < G2 ? __ldcg(p.part + (size_t)q * stride + kMlaHeads + h) : 0.f;
      }
      float M = -INFINITY;
#pragma unroll
      for (int j = 0; j < 5; ++j) M = fmaxf(M, mv[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int q = lane + 32 * j;
        if (q < G2) {
          const float w = mv[j] == -INFINITY ? 0.f : exp2f(mv[j] - M);
          wq[warp * G2 + q] = w;
          l = fmaf(lv[j], w, l);
        }
      }
      l = warp_allsum(l);
      if (lane == 0) wq[2 * G2 + warp] = 1.0f / l;
    }
    consumer_sync();
    mla_stamp(p, 14, tid);
    // element-parallel: thread (ei, qg) sums partials q = qg (mod 4) of element
    // e0 + ei, so a warp's load reads 32 consecutive floats of ONE partial
    // (coalesced; lanes over partials would cost one L2 sector per lane), 8
    // loads in flight per thread; the 4 q-subsets are added in fixed order
    float* zred = reinterpret_cast<float*>(zs) + 1024;  // [4][64], past wq
    const int ei = tid & 63, qg = tid >> 6;
    for (int eb = e0; eb < e1; eb += 64) {
      const int e = eb + ei;
      float acc = 0.f;
      if (e < e1) {
        const float* wrow = wq + (e / 512 - h0) * G2;
        for (int q0 = qg; q0 < G2; q0 += 32) {
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int q = q0 + 4 * j;
            v[j] = q < G2 ? __ldcg(p.part + (size_t)q * stride + 2 * kMlaHeads + e) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (q0 + 4 * j < G2) acc = fmaf(v[j], wrow[q0 + 4 * j], acc);
        }
      }
      zred[qg * 64 + ei] = acc;
      consumer_sync();
      if (tid < 64 && eb + tid < e1) {
        const float v = ((zred[tid] + zred[64 + tid]) + zred[128 + tid]) + zred[192 + tid];
        zloc[eb - e0 + tid] = round_to<__half>(v * wq[2 * G2 + (eb + tid) / 512 - h0]);
      }
      consumer_sync();
    }
  }
  mla_stamp(p, 9, tid);
  // 2. split-K share of o[h] = z[h] W_down[h] over this CTA's z elements: a
  //    warp's lanes own 4 of the H outputs, rows (z elements) come from the
  //    ring; warps are summed in order, then one fixed-point red.add per output
  int cnt = 0;
  float* wred = reinterpret_cast<float*>(zs) + 2560;  // [8 warps][H]
  for (int s = 0; s < 2; ++s) {
    const int h = eseg(s, ea, eb);
    if (s == 1 && h1 == h0) break;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int c4 = 4 * lane;  // this lane's outputs (H <= 128)
    consume_phase(s == 0 ? PD0 : PD1, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
      for (int r = 0; r < it.nunits; ++r) {
        const float z = zloc[ea + it.unit0 + r - e0];
        if (c4 < H) {
          const uint2 wv = *reinterpret_cast<const uint2*>(slot + (size_t)r * H * 2 + c4 * 2);
          const float2 w01 = __half22float2(*reinterpret_cast<const __half2*>(&wv.x));
          const float2 w23 = __half22float2(*reinterpret_cast<const __half2*>(&wv.y));
          acc[0] = fmaf(z, w01.x, acc[0]);
          acc[1] = fmaf(z, w01.y, acc[1]);
          acc[2] = fmaf(z, w23.x, acc[2]);
          acc[3] = fmaf(z, w23.y, acc[3]);
        }
      }
    });
    if (c4 < H) *reinterpret_cast<float4*>(wred + warp * 128 + c4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    consumer_sync();
    if (tid < H) {
      float v = 0.f;
      for (int w = 0; w < kNumConsumerWarps; ++w) v += wred[w * 128 + tid];
      red_add_fixed(p.o_acc + (size_t)h * H + tid, v);
    }
    consumer_sync();
  }
  mla_stamp(p, 11, tid);
  grid_barrier(p.barrier + 1, tid);
  mla_stamp(p, 12, tid);
  for (int t = tid; t < NH * H; t += kConsumerThreads)
    os[t] = __float2half_rn(fixed_to_float(__ldcg(p.o_acc + t)));
  consumer_sync();
  // 3. out = sum_h o[h] W_out[h] -> fixed point (each row owned by one CTA)
  tiled_gemv_phase<__half, 1, true>(PO, ring, warp, lane, tid, cnt, os, NH * H, 1,
                                    4 * (o1 - o0), part, [&](int row, int, float v) {
                                      p.accum[4 * o0 + row] = static_cast<unsigned long long>(
                                          __float2ll_rn(v * 4294967296.0f));
                                    });
  consumer_sync();
  mla_stamp(p, 13, tid);
}

// ------------------------------------------------------------------ host
template <class K>
static int launch_k(K kern, int grid, int block, size_t smem, bool pdl, const MlaEngParams& p,
                    cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return CFB_OK;
}

int mla_engine_decode(const cfb_mla_engine_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->n_heads < 1 || a->n_heads > kMlaHeads || a->kv_rank != 512 || a->head_dim % 8 || a->head_dim > 128 ||
      a->hidden % 512)
    return set_error(CFB_ERR_DIMENSION,
                     "head-batched MLA engine: 1..16 heads, kv_lora_rank 512, head_dim <= 128 (x8), hidden % 512 == 0");
  if (a->seq_len < 0) return set_error(CFB_ERR_DIMENSION, "seq_len must be >= 0");
  if (!a->resid || !a->norm_w || !a->w_a || !a->w_up || !a->w_dn || !a->w_o || !a->qc || !a->qlat ||
      !a->part || !a->o_acc || !a->accum || !a->barrier || (a->seq_len && !a->cache))
    return set_error(CFB_ERR_ARGUMENT, "null pointer");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  for (const auto& kc : {std::make_pair((const void*)mla_proj_kernel, kMaxSmem),
                         std::make_pair((const void*)mla_out_kernel, kMaxSmem),
                         std::make_pair((const void*)mla_attn_kernel, (int)kAttnSmem)})
    if (const int rc = configure_kernel(kc.first, kc.second, false)) return rc;
  MlaEngParams p = {};
  p.D = a->hidden;
  p.H = a->head_dim;
  p.NH = a->n_heads;
  p.R = a->kv_rank;
  p.S = a->seq_len;
  p.flags = a->flags;
  p.sleep_max = tuned_sleep();
  p.eps = a->eps;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)a->kv_rank));
  p.resid = a->resid;
  p.norm_w = static_cast<const __half*>(a->norm_w);
  p.w_a = static_cast<const __half*>(a->w_a);
  p.w_up = static_cast<const __half*>(a->w_up);
  p.w_dn = static_cast<const __half*>(a->w_dn);
  p.w_o = static_cast<const __half*>(a->w_o);
  p.cache = static_cast<const __half*>(a->cache);
  p.qc = static_cast<__half*>(a->qc);
  p.qlat = static_cast<__half*>(a->qlat);
  p.part = a->part;
  p.o_acc = a->o_acc;
  p.accum = a->accum;
  p.barrier = a->barrier;
  p.trace = a->trace;
  const int T = a->seq_len + 1;
  int G2 = (T + 63) / 64;
  if (G2 <= 20) G2 = (T + 31) / 32;  // short contexts: 32-row CTAs, the attention is latency-bound
  if (G2 > sms) G2 = sms;
  if (a->max_parts > 0 && G2 > a->max_parts) G2 = a->max_parts;
  if (G2 > 160) G2 = 160;  // mla_out_kernel's merge holds <= 5 partials per lane
  p.G2 = G2;
  const bool pdl = a->flags & CFB_PDL;
  int spw = tuned_spw();
  const int G = sms;
  // short contexts: the projection leaves the attention CTAs their own SMs, so
  // they are resident (streaming their cache rows) before the projection ends
  const int Gp = (G2 <= 72 && sms - G2 >= 64) ? sms - G2 : sms;
  while (spw > 1 && (mla_proj_layout(p.D, p.H, Gp, spw).total > kMaxSmem ||
                     mla_out_layout(p.D, p.H, G, spw).total > kMaxSmem))
    --spw;
  p.spw = spw;
  int rc = launch_k(mla_proj_kernel, Gp, kThreads, mla_proj_layout(p.D, p.H, Gp, spw).total, pdl, p, st);
  if (rc) return rc;
  if ((rc = launch_k(mla_attn_kernel, G2, kAttnThreads, kAttnSmem, true, p, st))) return rc;
  return launch_k(mla_out_kernel, G, kThreads, mla_out_layout(p.D, p.H, G, spw).total, true, p, st);
}

}  // namespace cfb
