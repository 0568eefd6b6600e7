// QKV projection of the attention module on ALL SMs (decode-engine split mode).
//
// The split_token cluster kernel runs n_heads x N CTAs (Llama2-7B: 32 x 4 =
// 128 of the 148 SMs) and with one CTA per SM its weight stream is capped by
// those SMs' in-flight bytes (~40 GB/s each).  The QKV rows are 75 % of the
// module's weight bytes, so this persistent kernel streams them over every SM
// (row-tiled GEMV, RMSNorm prologue, the same TMA-bulk ring as the FFN) and
// writes the fp16 q|k|v slices in the w_qkv row order; the cluster kernel
// (CFB_QKV_IN) then starts directly at the DSMEM gather.
#include <cuda_runtime.h>

#include "common.h"
#include "gemv.cuh"

namespace cfb {

struct QkvParams {
  int B, D, rows, spw, sleep_max;
  float eps;
  const float* resid;
  const __half* norm_w;
  const __half* w;   // row tiles [rows/4][D/8][4][8]
  __half* out;       // [B][rows]
};

__host__ __device__ inline int qkv_smem(int B, int D, int rows, int G, int spw, int* part_off) {
  const int tpc = (rows / 4 + G - 1) / G;
  int o = ring_bytes(spw) + 2 * kNumSlots * 8;
  const int xs = o;
  o += (B * D * 2 + 15) & ~15;
  *part_off = o;
  o += kNumConsumerWarps * B * 4 * tpc * 4;
  o += kNumConsumerWarps * B * 4;  // rmsnorm partials
  (void)xs;
  return o;
}

template <int QB>
__global__ void __launch_bounds__(kThreads, 1) qkv_proj_kernel(const QkvParams p) {
  extern __shared__ __align__(128) char smem[];
  const int G = gridDim.x, i = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int part_off;
  const int total = qkv_smem(p.B, p.D, p.rows, G, p.spw, &part_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes(p.spw));
  const Ring ring{smem, bars, bars + kNumSlots, p.spw, p.sleep_max};
  const int T = p.rows / 4;
  const int t0 = (int)((long long)i * T / G), t1 = (int)((long long)(i + 1) * T / G);
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const Phase P = make_phase(p.w + (size_t)t0 * 4 * p.D, nullptr, t1 - t0, 4 * p.D * 2, true);
  pdl_launch_dependents();
  if (warp == kNumConsumerWarps) {
    const Phase ph[1] = {P};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  pdl_wait();
  __half* xs = reinterpret_cast<__half*>(smem + ring_bytes(p.spw) + 2 * kNumSlots * 8);
  float* part = reinterpret_cast<float*>(smem + part_off);
  float* red = reinterpret_cast<float*>(smem + total - kNumConsumerWarps * p.B * 4);
  rmsnorm_to_smem<__half, true>(xs, p.resid, p.norm_w, p.B, p.D, p.eps, red, tid);
  int cnt = 0;
  const int rows = 4 * (t1 - t0);
  tiled_gemv_phase<__half, QB, true>(P, ring, warp, lane, tid, cnt, xs, p.D, p.B, rows, part,
                                     [&](int row, int b, float v) {
                                       p.out[(size_t)b * p.rows + 4 * t0 + row] = __float2half_rn(v);
                                     });
}

int qkv_proj(int dtype, int B, int D, int rows, const float* resid, const void* norm_w, float eps,
             const void* w, void* out, int flags, cudaStream_t st) {
  if (dtype != CFB_F16) return set_error(CFB_ERR_DIMENSION, "qkv_proj: fp16 only");
  if (B < 1 || B > 4 || D % 8 || rows % 4) return set_error(CFB_ERR_DIMENSION, "qkv_proj: bad shape");
  if (!resid || !norm_w || !w || !out) return set_error(CFB_ERR_ARGUMENT, "qkv_proj: null pointer");
  int dev = 0, sms = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  CFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int G = sms < rows / 4 ? sms : rows / 4;
  int spw = tuned_spw(), part_off = 0;
  while (spw > 1 && qkv_smem(B, D, rows, G, spw, &part_off) > kMaxSmem) --spw;
  const int smem = qkv_smem(B, D, rows, G, spw, &part_off);
  QkvParams p;
  p.B = B;
  p.D = D;
  p.rows = rows;
  p.spw = spw;
  p.sleep_max = tuned_sleep();
  p.eps = eps;
  p.resid = resid;
  p.norm_w = static_cast<const __half*>(norm_w);
  p.w = static_cast<const __half*>(w);
  p.out = static_cast<__half*>(out);
  auto launch = [&](auto kern) -> int {
    static bool configured = false;
    if (!configured) {
      CFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
      configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    LaunchAttrs at(0, flags & CFB_PDL);
    cfg.attrs = at.a;
    cfg.numAttrs = at.n;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
    return CFB_OK;
  };
  if (B == 1) return launch(qkv_proj_kernel<1>);
  if (B == 2) return launch(qkv_proj_kernel<2>);
  return launch(qkv_proj_kernel<4>);
}

}  // namespace cfb

extern "C" int cfb_qkv_proj(int dtype, int batch, int hidden, int rows, const float* resid,
                            const void* norm_w, float eps, const void* w_qkv, void* out, int flags,
                            void* stream) {
  return cfb::qkv_proj(dtype, batch, hidden, rows, resid, norm_w, eps, w_qkv, out, flags,
                       static_cast<cudaStream_t>(stream));
}
