// Batch-16 decode attention over INDEPENDENT sequences (BASELINE config #5
// "batch 16"): every sequence has its own KV cache and position, so - unlike
// the reference's shared-cache batch (oracle.py:45-50), which the cluster
// kernels keep for parity - the KV bytes grow with the batch and the kernel
// is a pure KV-streaming problem.  Split-KV flash decoding:
//
//   batch_attn_kernel  grid (chunk, sequence x head): 4 warps stream a
//                      256-position chunk of K (one 256 B row per warp load,
//                      4 positions in flight per warp) into scores, then the
//                      chunk softmax, then P V with one output dim per thread;
//                      partial (m, l, acc[128]) per chunk
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
  __shared__ float sc[kBaChunk];
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
  // scores: lane l covers dims 4l..4l+3 of a row; 4 rows per warp in flight
  const float q0 = qs[4 * lane], q1 = qs[4 * lane + 1], q2 = qs[4 * lane + 2], q3 = qs[4 * lane + 3];
  for (int r0 = p0 + 4 * warp; r0 < p1; r0 += 16) {
    uint2 kv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = min(r0 + j, p1 - 1);
      kv[j] = __ldg(reinterpret_cast<const uint2*>(K + (size_t)r * 128) + lane);
    }
    float d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&kv[j].x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&kv[j].y));
      d[j] = fmaf(q3, b.y, fmaf(q2, b.x, fmaf(q1, a.y, q0 * a.x)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] += __shfl_xor_sync(0xffffffffu, d[j], o);
    if (lane < 4 && r0 + lane < p1) sc[r0 + lane - p0] = d[lane] * scale;
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
  __syncthreads();
  // P V: thread = output dim, 8 rows in flight
  float acc = 0.f;
  int r = 0;
  for (; r + 8 <= n_rows; r += 8) {
    __half v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = V[(size_t)(p0 + r + j) * 128 + tid];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = fmaf(sc[r + j], __half2float(v[j]), acc);
  }
  for (; r < n_rows; ++r) acc = fmaf(sc[r], __half2float(V[(size_t)(p0 + r) * 128 + tid]), acc);
  if (tid == 0) {
    out[0] = m;
    out[1] = red[4] + red[5] + red[6] + red[7];
  }
  out[2 + tid] = acc;
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
