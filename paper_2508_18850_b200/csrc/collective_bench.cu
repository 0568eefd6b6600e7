// ClusterReduce / ClusterGather latency, on-chip (DSMEM) vs off-chip (global
// memory / L2): the B200 re-measurement of the paper's Table 1
// (the H100 numbers are the reference's
// fixtures/table1.csv:4-19).
//
// One cluster of N CTAs (256 threads each).  Operands and results live in
// shared memory, as in a fused kernel: every rank produces its data in smem
// (reduce: `bytes` of fp16 per rank, summed elementwise; gather: bytes / N per
// rank, concatenated in rank order) and consumes the result from smem.  The
// collective runs chunk by chunk, double-buffered:
//   on-chip : every rank pushes its chunk into each peer's receive slot with
//             ONE bulk DSMEM copy per peer (cp.async.bulk shared::cta ->
//             shared::cluster, completing on the peer's mbarrier), waits for
//             its own mbarrier, consumes; a relaxed cluster barrier arrive /
//             wait pair gives the senders back-pressure on the slots;
//   off-chip: every rank stores its chunk into a global scratch slot, the
//             ranks meet at a global-memory counter (red.release /
//             ld.acquire), then read the peers' slots back through L2.
// Reduce sums in fixed rank order with fp32 accumulation.  validate = 1 reads
// the operands from `in` and writes the results to `out` (tests); validate = 0
// (timing) computes the operands in registers and folds the results into a
// checksum, so no HBM traffic is timed.  `reps` collectives run back to back
// in one launch; rank 0 reports the mean globaltimer ns per collective.
#include "common.h"
#include "ptx.cuh"

namespace cfb {

namespace {

constexpr int kBenchThreads = 256;
constexpr int kStageBudget = 200 * 1024;  // smem for the double-buffered slots

__device__ __forceinline__ void add_h8(float (&acc)[8], const uint4& v) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __half22float2(h[j]);
    acc[2 * j] += f.x;
    acc[2 * j + 1] += f.y;
  }
}

__device__ __forceinline__ uint4 pack_h8(const float (&acc)[8]) {
  uint4 v;
  __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2half2_rn(acc[2 * j], acc[2 * j + 1]);
  return v;
}

__device__ __forceinline__ uint4 synth(int rank, int k, int v) {  // timing-mode operand
  const unsigned x = (unsigned)(rank * 0x9E3779B1u) ^ (unsigned)(k * 0x85EBCA77u) ^ (unsigned)v;
  return make_uint4(x & 0x3bff3bffu, (x >> 1) & 0x3bff3bffu, (x >> 2) & 0x3bff3bffu, (x >> 3) & 0x3bff3bffu);
}

// one bulk copy of `bytes` from this CTA's smem into CTA `dst`'s smem at the
// same offset as `local_dst`, completing on dst's copy of `local_bar`
__device__ __forceinline__ void dsmem_bulk_push(const void* src, void* local_dst, uint64_t* local_bar,
                                                uint32_t bytes, uint32_t dst) {
  const uint32_t raddr = mapa(smem_u32(local_dst), dst), rbar = mapa(smem_u32(local_bar), dst);
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          raddr),
      "r"(smem_u32(src)), "r"(bytes), "r"(rbar)
      : "memory");
}

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}

// N ranks meet at a monotonic global counter (the off-chip channel's barrier)
__device__ __forceinline__ void global_meet(unsigned long long* ctr, unsigned long long target) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_acquire_u64(ctr) < target) {
    }
  }
  __syncthreads();
}

// smem layout: bars[2] | slots[2][N][C]  (slot [b][q] = rank q's chunk)
template <bool kGather, bool kOnChip>
__global__ void __launch_bounds__(kBenchThreads, 1)
    collective_bench_kernel(int bytes, int chunk, int reps, int validate, const __half* in, __half* out,
                            __half* scratch, unsigned long long* ctr, unsigned long long* ns_out) {
  extern __shared__ __align__(128) char smem[];
  const int N = (int)cluster_nctas(), r = (int)cluster_rank(), tid = threadIdx.x;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* slots = smem + 128;
  const int contrib = kGather ? bytes / N : bytes;  // bytes each rank owns
  const int nchunks = (contrib + chunk - 1) / chunk;
  auto slot = [&](int b, int q) { return slots + ((size_t)b * N + q) * chunk; };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  // off-chip counter base: read before the start barrier, i.e. before any increment
  unsigned long long epoch = kOnChip ? 0ull : ld_acquire_u64(ctr) / N;
  __syncthreads();
  cluster_arrive();
  cluster_wait();
  uint32_t chk = 0;
  const unsigned long long t0 = globaltimer();
  int use = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int k = 0; k < nchunks; ++k, ++use) {
      const int b = use & 1;
      const int off = k * chunk, nb = min(chunk, contrib - off), nv = nb / 16;
      // 1. produce this rank's chunk into its own slot
      uint4* mine = reinterpret_cast<uint4*>(slot(b, r));
      for (int v = tid; v < nv; v += kBenchThreads)
        mine[v] = validate ? __ldg(reinterpret_cast<const uint4*>(in) + ((size_t)r * contrib + off) / 16 + v)
                           : synth(r, k, v);
      // 2. exchange
      if (kOnChip) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> bulk copy
        __syncthreads();
        if (use > 0) cluster_wait();  // peers consumed the previous chunk: slot b is free again
        if (tid == 0) {
          mbar_arrive_expect_tx(&bars[b], (uint32_t)((N - 1) * nb));
          for (int d = 1; d < N; ++d) dsmem_bulk_push(mine, mine, &bars[b], (uint32_t)nb, (uint32_t)((r + d) % N));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        mbar_wait(&bars[b], (use >> 1) & 1);
      } else {
        uint4* gs = reinterpret_cast<uint4*>(scratch) + ((size_t)b * N + r) * (chunk / 16);
        for (int v = tid; v < nv; v += kBenchThreads) __stcg(gs + v, mine[v]);
        ++epoch;
        global_meet(ctr, epoch * N);
        for (int q = 1; q < N; ++q) {
          const int src = (r + q) % N;
          const uint4* gq = reinterpret_cast<const uint4*>(scratch) + ((size_t)b * N + src) * (chunk / 16);
          uint4* dq = reinterpret_cast<uint4*>(slot(b, src));
          for (int v = tid; v < nv; v += kBenchThreads) dq[v] = __ldcg(gq + v);
        }
        __syncthreads();
      }
      // 3. consume the result from shared memory
      if (!kGather) {
        for (int v = tid; v < nv; v += kBenchThreads) {
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          for (int q = 0; q < N; ++q) add_h8(acc, reinterpret_cast<const uint4*>(slot(b, q))[v]);
          const uint4 o = pack_h8(acc);
          if (validate)
            reinterpret_cast<uint4*>(out)[((size_t)r * bytes + off) / 16 + v] = o;
          else
            chk += o.x ^ o.y ^ o.z ^ o.w;
        }
      } else {
        for (int e = tid; e < N * nv; e += kBenchThreads) {
          const int q = e / nv, v = e % nv;
          const uint4 x = reinterpret_cast<const uint4*>(slot(b, q))[v];
          if (validate)
            reinterpret_cast<uint4*>(out)[((size_t)r * bytes + (size_t)q * contrib + off) / 16 + v] = x;
          else
            chk += x.x ^ x.y ^ x.z ^ x.w;
        }
      }
      if (kOnChip) {
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // own slot reusable
        __syncthreads();
        cluster_arrive_relaxed();  // this rank is done with slot b (waited before the next push)
      }
    }
  }
  if (kOnChip && use > 0) cluster_wait();
  // no rank leaves while a peer may still address its smem
  cluster_arrive();
  cluster_wait();
  if (r == 0 && tid == 0) *ns_out = (globaltimer() - t0) / (unsigned long long)(reps > 0 ? reps : 1);
  if (!validate && chk == 0x12345678u) out[0] = __float2half(1.f);  // keep the consume alive
}

}  // namespace

int collective_bench(int op, int channel, int N, int bytes, int reps, int validate, const void* in, void* out,
                     void* scratch, unsigned long long* ctr, unsigned long long* ns_out, cudaStream_t st) {
  if (N < 2 || N > 16 || (N & (N - 1)))
    return set_error(CFB_ERR_CLUSTER_SIZE, "cluster size must be a power of two in [2, 16], got %d", N);
  if (op != 0 && op != 3) return set_error(CFB_ERR_ARGUMENT, "op must be 0 (reduce) or 3 (gather)");
  if (channel != 0 && channel != 1) return set_error(CFB_ERR_ARGUMENT, "channel must be 0 or 1");
  if (bytes < 16 * N || bytes % (16 * N) || reps < 1)
    return set_error(CFB_ERR_SHAPE, "bytes must be a positive multiple of 16 * N");
  if (!out || !ns_out || (validate && !in) || (channel == 1 && (!scratch || !ctr)))
    return set_error(CFB_ERR_ARGUMENT, "null buffer");
  // per-rank chunk: 2 buffers x N slots within the staging budget, <= 32 KB
  int chunk = kStageBudget / (2 * N);
  chunk = (chunk < 32768 ? chunk : 32768) & ~1023;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N, 1, 1);
  cfg.blockDim = dim3(kBenchThreads, 1, 1);
  cfg.dynamicSmemBytes = 128 + 2 * N * chunk;
  cfg.stream = st;
  LaunchAttrs la(N, false);
  cfg.attrs = la.a;
  cfg.numAttrs = la.n;
  const bool g = op == 3, on = channel == 0;
  auto k = g ? (on ? collective_bench_kernel<true, true> : collective_bench_kernel<true, false>)
             : (on ? collective_bench_kernel<false, true> : collective_bench_kernel<false, false>);
  if (const int rc = configure_kernel((const void*)k, kMaxSmem, true)) return rc;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, k, bytes, chunk, reps, validate, static_cast<const __half*>(in),
                              static_cast<__half*>(out), static_cast<__half*>(scratch), ctr, ns_out));
  return CFB_OK;
}

int collective_bench_chunk(int N) {
  int chunk = kStageBudget / (2 * N);
  return (chunk < 32768 ? chunk : 32768) & ~1023;
}

}  // namespace cfb
