// Batch-16 decode attention over INDEPENDENT sequences (BASELINE config #5
// "batch 16"): every sequence has its own KV cache and position, so - unlike
// the reference's shared-cache batch (oracle.py:45-50), which the cluster
// kernels keep for parity - the KV bytes grow with the batch and the kernel
// is a pure KV-streaming problem.  Split-KV flash decoding:
//
//   batch_attn_kernel  grid (128-position chunk, sequence x head): the chunk's
//                      K and V rows arrive by two bulk copies issued up front;
//                      scores, chunk softmax and P V from shared memory;
//                      partial (m, l, acc[128]) per chunk; the last chunk CTA
//                      of a (sequence, head) merges the partials and writes
//                      the head output in the packed UMMA activation layout
//                      of the O projection (cfb_tc_gemm_b16)
// Layouts: q [16][nh*128] fp16; caches [16][nh][cap][128] fp16; pos[16] = index
// of the newest (just appended) row, i.e. the sequence attends rows 0..pos.
#include <cuda_runtime.h>

#include "common.h"
#include "ptx.cuh"

namespace cfb {

constexpr int kBaChunk = 128;
static_assert(kBaChunk == CFB_KV_PAGE, "a KV page is one attention chunk");
constexpr int kBaThreads = 128;
// K, V chunk buffers, q, scores, P V row-lane partials, bars
constexpr int kBaSmem = 2 * kBaChunk * 256 + 2 * 128 * 4 + 8 * 128 * 4 + 64;
// chunks per CTA: a CTA walks cpc consecutive chunks of its (sequence, head),
// refilling the K buffer with the next chunk as soon as the scores are done
// and the V buffer as soon as P V is done, so its copies stay in flight while
// it computes (instead of draining at every chunk's CTA exit).  The host picks
// the largest power of two cpc <= kBaCpcMax for which the CTAs with a full
// cpc chunks still make >= 2 waves (same-box A/B: cpc 1 -> 2 -> 4/8 is
// 4.54 -> 4.33 -> 4.30 ms at 1K, 25.4 -> 23.0 -> 21.6 ms at 16K, batch 16).
constexpr int kBaCpcMax = 8;
constexpr int kBaCtasPerSm = 3;

// grid (chunk group, sequence x head).  Thread 0 issues a chunk's K rows and
// V rows as two bulk copies (64 KB in flight per CTA, 3 CTAs per SM); scores
// start when K lands, P V when V lands; the chunks of a CTA are combined
// online ((m, l, acc) rescaled per chunk).  Shared-memory reads are
// half-warp-per-256 B-row (conflict-free).  The last CTA of a (sequence,
// head) pair (ticket) merges the pair's partials and writes the head output
// as fp16 straight into the packed UMMA activation layout of the O projection.
__global__ void __launch_bounds__(kBaThreads) batch_attn_kernel(const __half* q, const __half* kc,
                                                                const __half* vc, const int* pos,
                                                                int nh, int cap, int nchunks, int kCpc,
                                                                float scale, float* part, int* ticket,
                                                                __half* xp, const int* table, int maxp) {
  extern __shared__ __align__(128) char smem[];
  __half* ks = reinterpret_cast<__half*>(smem);
  __half* vs = ks + kBaChunk * 128;
  float* qs = reinterpret_cast<float*>(vs + kBaChunk * 128);
  float* sc = qs + 128;
  float* pv = sc + 128;  // [8][128] P V row-lane partials
  uint64_t* bar = reinterpret_cast<uint64_t*>(pv + 8 * 128);
  __shared__ float red[8];
  __shared__ int last;
  // pos and the block table are set before the step (stable across its
  // kernels), and cache rows other than the new one were written by earlier
  // steps: the first chunk streams before griddepcontrol.wait unless it holds
  // the row the QKV projection is appending
  const int pair = blockIdx.y, n = pair / nh, h = pair % nh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = pos[n] + 1;
  // nused <= the launched chunks even for a position past max_len (the host
  // rejects that; the clamp keeps the merge ticket consistent regardless)
  const int nused = min((L + kBaChunk - 1) / kBaChunk, nchunks);
  // this sequence's chunks split evenly over nparts = ceil(nused / cpc) CTAs
  const int nparts = (nused + kCpc - 1) / kCpc;
  if ((int)blockIdx.x >= nparts) return;  // beyond this sequence: not part of its merge
  const int cb = (int)((long long)blockIdx.x * nused / nparts);
  const int nj = (int)((long long)(blockIdx.x + 1) * nused / nparts) - cb;
  auto rows_of = [&](int c) { return min(L, (c + 1) * kBaChunk) - c * kBaChunk; };
  // paged: chunk c of a sequence is exactly its page c (CFB_KV_PAGE == kBaChunk);
  // an unassigned entry (-1) reads page 0 instead of faulting (host-validated)
  auto base_of = [&](int c) -> size_t {
    if (table) return ((size_t)max(table[n * maxp + c], 0) * nh + h) * (size_t)kBaChunk * 128;
    return (((size_t)n * nh + h) * cap + (size_t)c * kBaChunk) * 128;
  };
  const uint64_t pol = policy_evict_first();
  auto issue_first = [&]() {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    const int r0 = rows_of(cb);
    const size_t b0 = base_of(cb);
    mbar_arrive_expect_tx(&bar[0], r0 * 256);
    bulk_g2s(ks, kc + b0, r0 * 256, &bar[0], pol);
    mbar_arrive_expect_tx(&bar[1], r0 * 256);
    bulk_g2s(vs, vc + b0, r0 * 256, &bar[1], pol);
  };
  const bool early = (cb + 1) * kBaChunk < L;  // the first chunk ends before the new row L - 1
  if (tid == 0 && early) issue_first();
  pdl_wait();
  pdl_launch_dependents();
  if (tid == 0 && !early) issue_first();
  qs[tid] = __half2float(q[(size_t)n * nh * 128 + h * 128 + tid]);
  __syncthreads();
  const int hl = lane & 15, ro = lane >> 4;
  float qv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) qv[e] = qs[8 * hl + e];
  float mrun = -INFINITY, lrun = 0.f, orun = 0.f;  // this CTA's chunks combined; orun: dimension tid
  for (int j = 0; j < nj; ++j) {
    const int c = cb + j, n_rows = rows_of(c);
    mbar_wait(&bar[0], j & 1);
    // scores: warp w covers rows w*32 .. +32, two rows per instruction, 4 in flight
#pragma unroll
    for (int r0 = 32 * warp; r0 < 32 * warp + 32; r0 += 8) {
      float d[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int r = min(r0 + 2 * jj + ro, n_rows - 1);
        const uint4 kv = reinterpret_cast<const uint4*>(ks + (size_t)r * 128)[hl];
        const __half2* hh = reinterpret_cast<const __half2*>(&kv);
        float t = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(hh[e]);
          t = fmaf(qv[2 * e + 1], f.y, fmaf(qv[2 * e], f.x, t));
        }
        d[jj] = t;
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) d[jj] += __shfl_xor_sync(0xffffffffu, d[jj], o);
      if (hl == 0)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) sc[r0 + 2 * jj + ro] = d[jj] * scale;
    }
    __syncthreads();
    if (tid == 0 && j + 1 < nj) {  // K buffer free: the next chunk's K rows
      const int rn = rows_of(c + 1);
      mbar_arrive_expect_tx(&bar[0], rn * 256);
      bulk_g2s(ks, kc + base_of(c + 1), rn * 256, &bar[0], pol);
    }
    // softmax over the chunk: thread = row
    const float sv = tid < n_rows ? sc[tid] : -INFINITY;
    float m = sv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float ev = tid < n_rows ? expf(sv - m) : 0.f;
    sc[tid] = ev;
    float l = ev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) red[4 + warp] = l;
    __syncthreads();
    // P V: thread = (row lane rl of 8, 8-dim group dg of 16)
    mbar_wait(&bar[1], j & 1);
    const int dg = tid & 15, rl = tid >> 4;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll 4
    for (int r = rl; r < n_rows; r += 8) {
      const uint4 v = reinterpret_cast<const uint4*>(vs + (size_t)r * 128)[dg];
      const float w = sc[r];
      const __half2* a = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(a[e]);
        acc[2 * e] = fmaf(w, f.x, acc[2 * e]);
        acc[2 * e + 1] = fmaf(w, f.y, acc[2 * e + 1]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) pv[rl * 128 + 8 * dg + e] = acc[e];
    __syncthreads();
    if (tid == 0 && j + 1 < nj) {  // V buffer free: the next chunk's V rows
      const int rn = rows_of(c + 1);
      mbar_arrive_expect_tx(&bar[1], rn * 256);
      bulk_g2s(vs, vc + base_of(c + 1), rn * 256, &bar[1], pol);
    }
    float accd = 0.f;
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) accd += pv[q2 * 128 + tid];
    const float lc = red[4] + red[5] + red[6] + red[7];
    if (j == 0) {
      mrun = m;
      lrun = lc;
      orun = accd;
    } else {  // online combine of the CTA's chunks
      const float M = fmaxf(mrun, m), a = expf(mrun - M), b = expf(m - M);
      lrun = fmaf(lc, b, lrun * a);
      orun = fmaf(accd, b, orun * a);
      mrun = M;
    }
  }
  float* out = part + ((size_t)pair * nchunks + blockIdx.x) * (2 + 128);
  if (tid == 0) {
    out[0] = mrun;
    out[1] = lrun;
  }
  out[2 + tid] = orun;
  // ticket: the last CTA of the pair merges
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int old = atomicAdd(ticket + pair, 1);
    last = old == nparts - 1;
    if (last) ticket[pair] = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* pp = part + (size_t)pair * nchunks * 130;
  // partial (m, l) loaded once, in parallel, into the (now free) K tile; every
  // thread then merges its dimension over the partials in order (the same
  // fmaf sequence as a serial merge), 8 partial loads in flight
  float* cm = reinterpret_cast<float*>(ks);  // [nparts] m, then the weights
  float* cl = cm + nchunks;                  // [nparts] l
  for (int cc = tid; cc < nparts; cc += kBaThreads) {
    cm[cc] = __ldcg(pp + (size_t)cc * 130);
    cl[cc] = __ldcg(pp + (size_t)cc * 130 + 1);
  }
  __syncthreads();
  float M = -INFINITY;
  for (int cc = 0; cc < nparts; ++cc) M = fmaxf(M, cm[cc]);
  __syncthreads();
  for (int cc = tid; cc < nparts; cc += kBaThreads) cm[cc] = expf(cm[cc] - M);
  __syncthreads();
  float lt = 0.f, at = 0.f;
  for (int c0 = 0; c0 < nparts; c0 += 8) {
    float a8[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) a8[jj] = c0 + jj < nparts ? __ldcg(pp + (size_t)(c0 + jj) * 130 + 2 + tid) : 0.f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
      if (c0 + jj < nparts) {
        lt = fmaf(cl[c0 + jj], cm[c0 + jj], lt);
        at = fmaf(a8[jj], cm[c0 + jj], at);
      }
  }
  // packed UMMA activation layout of nb rows (csrc/tc_gemm.cu xpack_off): K index h*128 + tid, row n
  const int nb = gridDim.y / nh, k = h * 128 + tid, kb = k / 64, kk = k % 64, s = kk / 16, c2 = (kk % 16) / 8;
  xp[(size_t)kb * (nb * 64) + ((s * 2 + c2) * (nb / 8) + n / 8) * 64 + (n % 8) * 8 + (kk % 8)] =
      __float2half_rn(__fdiv_rn(at, lt));
}

int batch_attention(const __half* q, const __half* kc, const __half* vc, const int* pos, int nh, int cap,
                    int max_len, float* part, int* ticket, __half* xp, const int* table, int maxp,
                    cudaStream_t st, bool pdl, int nb) {
  const int nchunks = (max_len + kBaChunk - 1) / kBaChunk;
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int cpc = 1;
  while (cpc < kBaCpcMax && (long long)nb * nh * (nchunks / (2 * cpc)) >= 2LL * kBaCtasPerSm * sms) cpc *= 2;
  auto kern = batch_attn_kernel;
  if (const int rc = configure_kernel((const void*)kern, kBaSmem, false)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((nchunks + cpc - 1) / cpc, nb * nh, 1);
  cfg.blockDim = dim3(kBaThreads, 1, 1);
  cfg.dynamicSmemBytes = kBaSmem;
  cfg.stream = st;
  LaunchAttrs at(0, pdl);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  const float scale = (float)(1.0 / std::sqrt(128.0));
  CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, q, kc, vc, pos, nh, cap, nchunks, cpc, scale, part, ticket,
                              xp, table, maxp));
  return CFB_OK;
}

// KV writer: grid (count, n_heads), 16 threads x 16 B per 256 B row
__global__ void kv_write_kernel(__half* kc, __half* vc, const int* table, int maxp, int cap, int nh, int seq,
                                int start, int count, const __half* ks, const __half* vs) {
  const int r = blockIdx.x, h = blockIdx.y, t = threadIdx.x, p = start + r;
  if (table && table[seq * maxp + p / kBaChunk] < 0) return;  // unassigned page
  const size_t dst = table ? (((size_t)table[seq * maxp + p / kBaChunk] * nh + h) * kBaChunk + p % kBaChunk) * 128
                           : (((size_t)seq * nh + h) * cap + p) * 128;
  const size_t src = ((size_t)h * count + r) * 128;
  reinterpret_cast<uint4*>(kc + dst)[t] = reinterpret_cast<const uint4*>(ks + src)[t];
  reinterpret_cast<uint4*>(vc + dst)[t] = reinterpret_cast<const uint4*>(vs + src)[t];
}

int kv_write(__half* kc, __half* vc, const int* table, int maxp, int cap, int nh, int seq, int start, int count,
             const __half* ks, const __half* vs, cudaStream_t st) {
  if (!kc || !vc || (count > 0 && (!ks || !vs)) || seq < 0 || seq >= 32 || start < 0 || count < 0 || nh <= 0)
    return set_error(CFB_ERR_ARGUMENT, "kv_write: bad arguments");
  if (!table && start + count > cap) return set_error(CFB_ERR_DIMENSION, "kv_write: rows beyond cache_cap");
  if (table && start + count > maxp * kBaChunk) return set_error(CFB_ERR_DIMENSION, "kv_write: rows beyond the block table");
  if (!count) return CFB_OK;
  kv_write_kernel<<<dim3(count, nh), 16, 0, st>>>(kc, vc, table, maxp, cap, nh, seq, start, count, ks, vs);
  CFB_CUDA(cudaGetLastError());
  return CFB_OK;
}

}  // namespace cfb

extern "C" int cfb_b16_kv_write(void* k_cache, void* v_cache, const int* block_table, int max_pages, int cache_cap,
                                int n_heads, int seq, int start, int count, const void* k_src, const void* v_src,
                                void* stream) {
  return cfb::kv_write(static_cast<__half*>(k_cache), static_cast<__half*>(v_cache), block_table, max_pages,
                       cache_cap, n_heads, seq, start, count, static_cast<const __half*>(k_src),
                       static_cast<const __half*>(v_src), static_cast<cudaStream_t>(stream));
}
