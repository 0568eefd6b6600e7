// split_head attention module (ClusterFusion App. B.2) for sm_100a.
//
// Mirrors reference dataflows.py:432-502 (run_splithead_decode), the
// head-dimension partition the paper compares split_token against
// (PAPER.md:1229-1234): one cluster of N CTAs per head, CTA rank r owns
// head-dim slice [r*h, (r+1)*h) of q, k and v throughout:
//   1. q_r, k_r, v_r = x @ W_qkv[head][:, slice]  (new token, kept in fp32
//      like the reference's python locals)                 dataflows.py:447-460
//   2. partial scores q_r . K[:, slice]^T * 1/sqrt(H) over all S (+B) keys,
//      store-rounded, SUM ClusterReduce -> full scores      :462-466
//   3. every CTA: softmax of the full scores, att_r = P @ V[:, slice],
//      out_r = att_r @ W_out[head][slice, :] (B x D), SUM ClusterReduce   :468-484
//   4. rank 0 adds the head's (B x D) output into the 64-bit fixed-point
//      cross-head accumulator                               :486-492
// This dataflow is latency/compute-secondary (its reduce payloads grow with
// S and D); it streams K/V/W with plain coalesced loads and keeps the score
// and output-projection buffers in shared memory (SmemOverflow when they do
// not fit, like the reference's smem_capacity_bytes check).
#include <cuda_runtime.h>

#include "collectives.cuh"
#include "common.h"

namespace cfb {

namespace {
constexpr int kShThreads = 256;

struct ShParams {
  int B, D, H, Hp, N, n_heads, S, att, flags;
  float scale;
  const void* x;       // [B][D]
  const void* w_qkv;   // [n_heads][D][3H] (reference layout)
  const void* w_out;   // [n_heads][H][D]  (reference layout)
  const void* k_cache; // [n_heads][S][H]
  const void* v_cache;
  unsigned long long* accum;
  float* stats;
  unsigned long long* traffic;
};

struct ShLayout {
  int bars, xs, qkv, sc, scrx, pr, op, oprx, total, sc_bytes, op_bytes;
};

__host__ __device__ inline int rnd16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline ShLayout sh_layout(int B, int D, int H, int att, int N, int tb) {
  ShLayout L;
  const int h = H / N;
  L.sc_bytes = rnd16(B * att * tb);
  L.op_bytes = rnd16(B * D * tb);
  int o = 0;
  L.bars = o;  o += 8 * 8;
  L.xs = o;    o += rnd16(B * D * 4);
  L.qkv = o;   o += rnd16(4 * B * h * 4);  // q, k, v of the new token(s), then att
  L.sc = o;    o += L.sc_bytes;
  L.scrx = o;  o += 4 * L.sc_bytes;
  L.pr = o;    o += rnd16(B * att * 4) + rnd16(2 * B * 4);
  L.op = o;    o += L.op_bytes;
  L.oprx = o;  o += 4 * L.op_bytes;
  L.total = o;
  return L;
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(kShThreads, 1) splithead_kernel(const ShParams p) {
  extern __shared__ __align__(128) char smem[];
  constexpr int tb = sizeof(T);
  const int B = p.B, D = p.D, H = p.H, att = p.att;
  const uint32_t N = p.N;
  const int h = H / (int)N;
  const ShLayout L = sh_layout(B, D, H, att, N, tb);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + L.bars);  // [0,4) scores, [4,8) out_proj
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int head = blockIdx.y, lo = (int)rank * h;
  int rounds = 0;
  while ((1u << rounds) < N) ++rounds;
  if (tid == 0) {
    for (int r = 0; r < rounds; ++r) {
      mbar_init(&cbar[r], 1);
      mbar_arrive_expect_tx(&cbar[r], L.sc_bytes);
      mbar_init(&cbar[4 + r], 1);
      mbar_arrive_expect_tx(&cbar[4 + r], L.op_bytes);
    }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_arrive();

  float* xs = reinterpret_cast<float*>(smem + L.xs);
  float* qkv = reinterpret_cast<float*>(smem + L.qkv);  // [3][B][h]
  T* sc = reinterpret_cast<T*>(smem + L.sc);
  float* pr = reinterpret_cast<float*>(smem + L.pr);    // probabilities [B][att], then m, l
  float* ml = pr + (rnd16(B * att * 4) / 4);
  T* op = reinterpret_cast<T*>(smem + L.op);
  const T* X = static_cast<const T*>(p.x);
  const T* W = static_cast<const T*>(p.w_qkv) + (size_t)head * D * 3 * H;
  const T* Wo = static_cast<const T*>(p.w_out) + (size_t)head * H * D;
  const T* Kc = static_cast<const T*>(p.k_cache) + (size_t)head * p.S * H;
  const T* Vc = static_cast<const T*>(p.v_cache) + (size_t)head * p.S * H;

  for (int i = tid; i < B * D; i += kShThreads) xs[i] = Elem<T>::to_f(X[i]);
  __syncthreads();
  // 1. q/k/v slices of the new token(s): one warp per output, lanes over D
  for (int o = warp; o < 3 * B * h; o += kShThreads / 32) {
    const int which = o / (B * h), b = (o / h) % B, i = o % h;
    const int col = which * H + lo + i;
    float s = 0.f;
    for (int d = lane; d < D; d += 32) s = fmaf(xs[b * D + d], Elem<T>::to_f(W[(size_t)d * 3 * H + col]), s);
    for (int k = 16; k > 0; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
    if (lane == 0) qkv[o] = s;
  }
  __syncthreads();
  const float* qn = qkv;
  const float* kn = qkv + B * h;
  const float* vn = qkv + 2 * B * h;
  // 2. partial scores over this rank's head-dim slice
  for (int idx = tid; idx < B * att; idx += kShThreads) {
    const int b = idx / att, j = idx % att;
    float s = 0.f;
    for (int i = 0; i < h; ++i) {
      const float k = j < p.S ? Elem<T>::to_f(Kc[(size_t)j * H + lo + i]) : kn[(j - p.S) * h + i];
      s = fmaf(qn[b * h + i], k, s);
    }
    sc[idx] = Elem<T>::from_f(__fmul_rn(s, p.scale));
  }
  for (int idx = B * att + tid; idx < L.sc_bytes / tb; idx += kShThreads) sc[idx] = Elem<T>::from_f(0.f);
  __syncthreads();
  cluster_wait();  // peers' mbarriers initialised
  unsigned long long sent_sc = 0, sent_op = 0;
  if (warp == 0) {
    T* rx[4];
    uint64_t* rb[4];
    for (int r = 0; r < 4; ++r) {
      rx[r] = reinterpret_cast<T*>(smem + L.scrx + r * L.sc_bytes);
      rb[r] = &cbar[r];
    }
    warp_cluster_reduce<T>(sc, B * att, L.sc_bytes, rx, rb, kSum, rank, N, lane);
    for (int r = 0; r < rounds; ++r) sent_sc += (unsigned long long)B * att * tb;
  }
  __syncthreads();
  // 3. softmax of the full scores (every CTA), att = P @ V[:, slice]
  if (warp < B) {
    const int b = warp;
    float m = -INFINITY;
    for (int j = lane; j < att; j += 32) m = fmaxf(m, Elem<T>::to_f(sc[b * att + j]));
    for (int k = 16; k > 0; k >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, k));
    float l = 0.f;
    for (int j = lane; j < att; j += 32) {
      const float w = expf(Elem<T>::to_f(sc[b * att + j]) - m);
      pr[b * att + j] = w;
      l += w;
    }
    for (int k = 16; k > 0; k >>= 1) l += __shfl_xor_sync(0xffffffffu, l, k);
    if (lane == 0) {
      ml[2 * b] = m;
      ml[2 * b + 1] = l;
    }
  }
  __syncthreads();
  float* at = qkv + 3 * B * h;  // att [B][h] = (P / l) @ V[:, slice]
  for (int o = warp; o < B * h; o += kShThreads / 32) {
    const int b = o / h, i = o % h;
    float s = 0.f;
    for (int j = lane; j < att; j += 32) {
      const float v = j < p.S ? Elem<T>::to_f(Vc[(size_t)j * H + lo + i]) : vn[(j - p.S) * h + i];
      s = fmaf(__fdiv_rn(pr[b * att + j], ml[2 * b + 1]), v, s);
    }
    for (int k = 16; k > 0; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
    if (lane == 0) at[o] = s;
  }
  __syncthreads();
  // out_r = att_r @ W_out[head][slice, :]
  for (int idx = tid; idx < B * D; idx += kShThreads) {
    const int b = idx / D, c = idx % D;
    float s = 0.f;
    for (int i = 0; i < h; ++i) s = fmaf(at[b * h + i], Elem<T>::to_f(Wo[(size_t)(lo + i) * D + c]), s);
    op[idx] = Elem<T>::from_f(s);
  }
  for (int idx = B * D + tid; idx < L.op_bytes / tb; idx += kShThreads) op[idx] = Elem<T>::from_f(0.f);
  __syncthreads();
  if (warp == 0) {
    T* rx[4];
    uint64_t* rb[4];
    for (int r = 0; r < 4; ++r) {
      rx[r] = reinterpret_cast<T*>(smem + L.oprx + r * L.op_bytes);
      rb[r] = &cbar[4 + r];
    }
    warp_cluster_reduce<T>(op, B * D, L.op_bytes, rx, rb, kSum, rank, N, lane);
    for (int r = 0; r < rounds; ++r) sent_op += (unsigned long long)B * D * tb;
    if (lane == 0 && p.traffic) {
      atomicAdd(&p.traffic[CFB_STAGE_SCORE_REDUCE], sent_sc);
      atomicAdd(&p.traffic[CFB_STAGE_OUT_PROJ_REDUCE], sent_op);
    }
    if (rank == 0 && p.stats)
      for (int b = lane; b < B; b += 32) {
        p.stats[((size_t)head * 2) * B + b] = ml[2 * b];
        p.stats[((size_t)head * 2 + 1) * B + b] = ml[2 * b + 1];
      }
  }
  __syncthreads();
  // 4. rank 0 writes the head output once
  if (rank == 0)
    for (int idx = tid; idx < B * D; idx += kShThreads) red_add_fixed(&p.accum[idx], Elem<T>::to_f(op[idx]));
  cluster_arrive();
  cluster_wait();
}

int splithead_decode(const cfb_splithead_args* a, cudaStream_t st) {
  if (!a) return set_error(CFB_ERR_ARGUMENT, "null args");
  if (a->dtype != CFB_F16 && a->dtype != CFB_F32)
    return set_error(CFB_ERR_ARGUMENT, "dtype must be CFB_F16 (2) or CFB_F32 (4)");
  const int N = a->cluster, tb = a->dtype;
  if (N < 1 || N > 16 || (N & (N - 1)))
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16], got %d", N);
  if (a->batch < 1 || a->batch > 8) return set_error(CFB_ERR_DIMENSION, "split_head batch must be in [1, 8]");
  if (a->head_dim % N)
    return set_error(CFB_ERR_DIMENSION, "head_dim %d not divisible by cluster size %d", a->head_dim, N);
  if (a->seq_len < 0) return set_error(CFB_ERR_DIMENSION, "seq_len must be >= 0");
  const int att = a->seq_len + ((a->flags & CFB_APPEND) ? a->batch : 0);
  if (att == 0) return set_error(CFB_ERR_DIMENSION, "no attended positions: empty cache and no appended token");
  if (!a->x || !a->w_qkv || !a->w_out || !a->accum || (a->seq_len && (!a->k_cache || !a->v_cache)))
    return set_error(CFB_ERR_ARGUMENT, "null input / weight / accumulator pointer");
  const ShLayout L = sh_layout(a->batch, a->hidden, a->head_dim, att, N, tb);
  if (L.total > kMaxSmem)
    return set_error(CFB_ERR_SMEM, "split_head needs %d B of shared memory per CTA (max %d)", L.total,
                     kMaxSmem);
  ShParams p;
  p.B = a->batch;
  p.D = a->hidden;
  p.H = a->head_dim;
  p.Hp = a->head_dim;
  p.N = N;
  p.n_heads = a->n_heads;
  p.S = a->seq_len;
  p.att = att;
  p.flags = a->flags;
  p.scale = (float)(1.0 / std::sqrt((double)a->head_dim));
  p.x = a->x;
  p.w_qkv = a->w_qkv;
  p.w_out = a->w_out;
  p.k_cache = a->k_cache;
  p.v_cache = a->v_cache;
  p.accum = a->accum;
  p.stats = a->stats;
  p.traffic = a->traffic;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N, a->n_heads, 1);
  cfg.blockDim = dim3(kShThreads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  LaunchAttrs at(N, false);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  if (tb == 2) {
    if (const int rc = configure_kernel((const void*)splithead_kernel<__half>, kMaxSmem, true)) return rc;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, splithead_kernel<__half>, p));
  } else {
    if (const int rc = configure_kernel((const void*)splithead_kernel<float>, kMaxSmem, true)) return rc;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, splithead_kernel<float>, p));
  }
  if (!a->out) return CFB_OK;
  return mha_finalize(a->out, nullptr, a->accum, a->batch * a->hidden, st);
}

}  // namespace cfb
