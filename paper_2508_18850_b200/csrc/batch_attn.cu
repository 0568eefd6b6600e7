// Batch-16 decode attention over INDEPENDENT sequences (BASELINE config #5
// "batch 16"): every sequence has its own KV cache and position, so - unlike
// the reference's shared-cache batch (oracle.py:45-50), which the cluster
// kernels keep for parity - the KV bytes grow with the batch and the kernel
// is a pure KV-streaming problem.  Split-KV flash decoding:
//
//   batch_attn_kernel  grid (chunk, sequence x head): 4 warps stream a
//                      256-position chunk of K (a half-warp per 256 B row,
//                      16 B per lane, 8 rows in flight per warp) into scores,
//                      then the chunk softmax, then P V with 16 B V loads
//                      (thread = 8 dims x a row lane, 2 rows in flight),
//                      summed over the row lanes in smem; partial
//                      (m, l, acc[128]) per chunk
//   batch_merge_kernel one CTA per (sequence, head): merges the chunk partials
//                      and writes the head output as fp16 straight into the
//                      packed UMMA activation layout of the O-projection
//                      (cfb_tc_gemm_b16)
// Layouts: q [16][nh*128] fp16; caches [16][nh][cap][128] fp16; pos[16] = index
// of the newest (just appended) row, i.e. the sequence attends rows 0..pos.
#include <cuda_runtime.h>

#include "common.h"
#include "ptx.cuh"

namespace cfb {

constexpr int kBaChunk = 256;
constexpr int kBaThreads = 128;

__global__ void __launch_bounds__(kBaThreads) batch_attn_kernel(const __half* q, const __half* kc,
                                                                const __half* vc, const int* pos,
                                                                int nh, int cap, int nchunks,
                                                                float scale, float* part) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ float qs[128];
  __shared__ float sc[kBaChunk > 1024 ? kBaChunk : 1024];  // scores, then 8 x 128 PV partials
  __shared__ float red[8];
  const int pair = blockIdx.y, n = pair / nh, h = pair % nh, c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = pos[n] + 1, p0 = c * kBaChunk, p1 = min(L, p0 + kBaChunk);
  float* out = part + ((size_t)pair * nchunks + c) * (2 + 128);
  if (p0 >= p1) {  // empty chunk: softmax identity
    if (tid == 0) {
      out[0] = -INFINITY;
      out[1] = 0.f;
    }
    out[2 + tid] = 0.f;
    return;
  }
  qs[tid] = __half2float(q[(size_t)n * nh * 128 + h * 128 + tid]);
  __syncthreads();
  const size_t base = ((size_t)n * nh + h) * cap * 128;
  const __half* K = kc + base;
  const __half* V = vc + base;
  // scores: half-warp per row (lane covers 8 dims = 16 B), 2 rows per warp load,
  // 4 loads (8 rows) in flight per warp
  const int hl = lane & 15, ro = lane >> 4;
  float qv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) qv[e] = qs[8 * hl + e];
  for (int r0 = p0 + 8 * warp; r0 < p1; r0 += 32) {
    uint4 kv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = min(r0 + 2 * j + ro, p1 - 1);
      kv[j] = __ldg(reinterpret_cast<const uint4*>(K + (size_t)r * 128) + hl);
    }
    float d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __half2* hh = reinterpret_cast<const __half2*>(&kv[j]);
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(hh[e]);
        t = fmaf(qv[2 * e + 1], f.y, fmaf(qv[2 * e], f.x, t));
      }
      d[j] = t;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] += __shfl_xor_sync(0xffffffffu, d[j], o);
    if (hl == 0)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + 2 * j + ro;
        if (r < p1) sc[r - p0] = d[j] * scale;
      }
  }
  __syncthreads();
  const int n_rows = p1 - p0;
  float m = -INFINITY;
  for (int r = tid; r < n_rows; r += kBaThreads) m = fmaxf(m, sc[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  float l = 0.f;
  for (int r = tid; r < n_rows; r += kBaThreads) {
    const float e = expf(sc[r] - m);
    sc[r] = e;
    l += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  __syncthreads();
  if (lane == 0) red[4 + warp] = l;
  // P V: thread = (row lane rl of 8, dim group dg of 16 x 8 dims), 16 B loads,
  // 2 rows in flight per thread; the 8 row lanes are summed through smem
  const int dg = tid & 15, rl = tid >> 4;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int r = rl; r < n_rows; r += 16) {
    const int r2 = min(r + 8, n_rows - 1);
    const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(V + (size_t)(p0 + r) * 128) + dg);
    const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(V + (size_t)(p0 + r2) * 128) + dg);
    const float w0 = sc[r], w1 = r + 8 < n_rows ? sc[r2] : 0.f;
    const __half2* a0 = reinterpret_cast<const __half2*>(&v0);
    const __half2* a1 = reinterpret_cast<const __half2*>(&v1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f0 = __half22float2(a0[e]), f1 = __half22float2(a1[e]);
      acc[2 * e] = fmaf(w1, f1.x, fmaf(w0, f0.x, acc[2 * e]));
      acc[2 * e + 1] = fmaf(w1, f1.y, fmaf(w0, f0.y, acc[2 * e + 1]));
    }
  }
  __syncthreads();  // sc no longer needed: reuse it for the row-lane partials
#pragma unroll
  for (int e = 0; e < 8; ++e) sc[rl * 128 + 8 * dg + e] = acc[e];
  __syncthreads();
  float accd = 0.f;
#pragma unroll
  for (int q2 = 0; q2 < 8; ++q2) accd += sc[q2 * 128 + tid];
  const float acc_out = accd;
  if (tid == 0) {
    out[0] = m;
    out[1] = red[4] + red[5] + red[6] + red[7];
  }
  out[2 + tid] = acc_out;
}

// one CTA (128 threads = head dims) per (sequence, head)
__global__ void __launch_bounds__(kBaThreads) batch_merge_kernel(const float* part, int nh, int nchunks,
                                                                 __half* xp) {
  pdl_wait();
  pdl_launch_dependents();
  const int pair = blockIdx.x, n = pair / nh, h = pair % nh, tid = threadIdx.x;
  const float* pp = part + (size_t)pair * nchunks * (2 + 128);
  float M = -INFINITY;
  for (int c = 0; c < nchunks; ++c) M = fmaxf(M, pp[(size_t)c * 130]);
  float l = 0.f, a = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const float mc = pp[(size_t)c * 130];
    const float w = mc == -INFINITY ? 0.f : expf(mc - M);
    l = fmaf(pp[(size_t)c * 130 + 1], w, l);
    a = fmaf(pp[(size_t)c * 130 + 2 + tid], w, a);
  }
  // packed UMMA activation layout (csrc/tc_gemm.cu): K index = h*128 + tid, row n
  const int k = h * 128 + tid, kb = k / 64, kk = k % 64, s = kk / 16, cc = (kk % 16) / 8;
  xp[(size_t)kb * 1024 + ((s * 2 + cc) * 2 + n / 8) * 64 + (n % 8) * 8 + (kk % 8)] = __float2half_rn(__fdiv_rn(a, l));
}

int batch_attention(const __half* q, const __half* kc, const __half* vc, const int* pos, int nh, int cap,
                    int max_len, float* part, __half* xp, cudaStream_t st, bool pdl) {
  const int nchunks = (max_len + kBaChunk - 1) / kBaChunk;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nchunks, 16 * nh, 1);
  cfg.blockDim = dim3(kBaThreads, 1, 1);
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  const float scale = (float)(1.0 / std::sqrt(128.0));
  CFB_CUDA(cudaLaunchKernelEx(&cfg, batch_attn_kernel, q, kc, vc, pos, nh, cap, nchunks, scale, part));
  cudaLaunchConfig_t c2 = cfg;
  c2.gridDim = dim3(16 * nh, 1, 1);
  LaunchAttrs at2(0, true);
  c2.attrs = at2.a;
  c2.numAttrs = at2.n;
  CFB_CUDA(cudaLaunchKernelEx(&c2, batch_merge_kernel, (const float*)part, nh, nchunks, xp));
  return CFB_OK;
}

}  // namespace cfb
