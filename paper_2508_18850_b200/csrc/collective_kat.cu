// Stand-alone ClusterReduce / ClusterGather kernel: one cluster of N CTAs,
// CTA r contributes in[r].  Used to port the reference's collective KATs
// (tests/test_collectives.py) onto the real DSMEM primitives.
#include "collectives.cuh"
#include "common.h"

namespace cfb {

template <typename T>
__global__ void collective_kat_kernel(int op, int n, const T* in, T* out,
                                      unsigned long long* traffic) {
  extern __shared__ __align__(128) char smem[];
  const uint32_t rank = cluster_rank(), N = cluster_nctas();
  const int lane = threadIdx.x;
  constexpr int tb = sizeof(T);
  const int seg_bytes = (n * tb + 15) & ~15;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* buf = smem + 128;                   // reduce buffer or gather buffer (N segments)
  char* rx = buf + N * seg_bytes;           // 4 receive slots (reduce)
  int rounds = 0;
  while ((1u << rounds) < N) ++rounds;
  if (lane == 0) {
    for (int r = 0; r < rounds; ++r) {
      mbar_init(&bars[r], 1);
      mbar_arrive_expect_tx(&bars[r], op == 3 ? (1u << r) * seg_bytes : seg_bytes);
    }
    fence_mbar_init();
  }
  for (int i = lane; i < N * seg_bytes / tb; i += 32) reinterpret_cast<T*>(buf)[i] = T(0);
  __syncwarp();
  for (int i = lane; i < n; i += 32) reinterpret_cast<T*>(buf)[i] = in[(size_t)rank * n + i];
  __syncwarp();
  cluster_arrive();
  cluster_wait();
  uint64_t* rb[4] = {&bars[0], &bars[1], &bars[2], &bars[3]};
  unsigned long long sent = 0;
  if (op == 3) {
    warp_cluster_gather(buf, seg_bytes, rb, rank, N, lane);
    for (uint32_t s = 1; s < N; s <<= 1) sent += (unsigned long long)s * n * tb;
    for (int i = lane; i < (int)N * n; i += 32) {
      const int j = i / n, k = i % n;
      out[(size_t)rank * N * n + i] = reinterpret_cast<T*>(buf + j * seg_bytes)[k];
    }
  } else {
    T* rxp[4] = {reinterpret_cast<T*>(rx), reinterpret_cast<T*>(rx + seg_bytes),
                 reinterpret_cast<T*>(rx + 2 * seg_bytes), reinterpret_cast<T*>(rx + 3 * seg_bytes)};
    warp_cluster_reduce<T>(reinterpret_cast<T*>(buf), n, seg_bytes, rxp, rb, op, rank, N, lane);
    sent = (unsigned long long)rounds * n * tb;
    for (int i = lane; i < n; i += 32) out[(size_t)rank * n + i] = reinterpret_cast<T*>(buf)[i];
  }
  if (lane == 0 && traffic) atomicAdd(traffic, sent);
  cluster_arrive();
  cluster_wait();
}

int cluster_collective(int dtype, int op, int N, int n, const void* in, void* out,
                       unsigned long long* traffic, cudaStream_t st) {
  if (N < 1 || N > 16 || (N & (N - 1)))
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [1, 16], got %d", N);
  if (op < 0 || op > 3) return set_error(CFB_ERR_ARGUMENT, "op must be 0..3");
  if (dtype != CFB_F16 && dtype != CFB_F32) return set_error(CFB_ERR_ARGUMENT, "bad dtype");
  if (op == 2 && (n % 2)) return set_error(CFB_ERR_SHAPE, "softmax_merge requires an even-length buffer");
  if (n < 1 || !in || !out) return set_error(CFB_ERR_ARGUMENT, "bad buffer");
  const int seg_bytes = (n * dtype + 15) & ~15;
  const size_t smem = 128 + (size_t)N * seg_bytes + 4 * seg_bytes;
  if (smem > (size_t)kMaxSmem) return set_error(CFB_ERR_SMEM, "payload too large");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N, 1, 1);
  cfg.blockDim = dim3(32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = N;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == CFB_F16) {
    auto k = collective_kat_kernel<__half>;
    if (const int rc = configure_kernel((const void*)k, kMaxSmem, true)) return rc;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, k, op, n, static_cast<const __half*>(in),
                                static_cast<__half*>(out), traffic));
  } else {
    auto k = collective_kat_kernel<float>;
    if (const int rc = configure_kernel((const void*)k, kMaxSmem, true)) return rc;
    CFB_CUDA(cudaLaunchKernelEx(&cfg, k, op, n, static_cast<const float*>(in),
                                static_cast<float*>(out), traffic));
  }
  return CFB_OK;
}

}  // namespace cfb
