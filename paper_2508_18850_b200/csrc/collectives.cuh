// DSMEM ClusterReduce / ClusterGather (ClusterFusion Alg. 1 / Alg. 2).
//
// Schedule (reference collectives.py:105-203): log2(N) rounds; in round r
// (stride s = 2^r) CTA b sends to (b + s) mod N and receives from
// (b - s) mod N.  Reduce keeps the message size constant and folds
// op(own, received) into the local buffer, rounding to the storage type at
// every store (simcore.py:94-110).  Gather forwards the already-assembled
// prefix of s segments, leaving the rank-rotated layout
// (segment j of CTA b holds rank (b - j) mod N).
//
// Transport: the sender pushes its message with st.async straight into a
// per-round receive slot in the peer's shared memory; every slot has its own
// mbarrier whose expected byte count the receiver posted at kernel start, so
// completion is signalled by the bytes themselves (no cluster-wide barrier,
// no acknowledgements: every slot is written exactly once per launch).
//
// All functions run on ONE full warp.
#pragma once
#include "ptx.cuh"

namespace cfb {

enum ReduceKind { kSum = 0, kMax = 1, kSoftmaxMerge = 2 };

// Push `bytes` (multiple of 16) from local smem `src` into CTA `dst`'s
// shared memory at the address that `local_dst` has locally, completing on
// the peer's copy of `local_bar`.
__device__ __forceinline__ void dsmem_push(const void* src, void* local_dst, uint64_t* local_bar,
                                           int bytes, uint32_t dst, int lane) {
  const uint32_t raddr = mapa(smem_u32(local_dst), dst);
  const uint32_t rbar = mapa(smem_u32(local_bar), dst);
  const char* s = static_cast<const char*>(src);
  for (int v = lane; v < bytes / 16; v += 32) st_async_v4(raddr + 16 * v, lds128(s + 16 * v), rbar);
}

// In-place all-reduce of `buf` (n logical elements, `bytes_pad` = padded
// buffer bytes) over the cluster.  rx[r] / rx_bar[r]: receive slot of round r.
// For kSoftmaxMerge the buffer is [m_0..m_{B-1} | l_0..l_{B-1}] with n = 2B.
template <typename T>
__device__ void warp_cluster_reduce(T* buf, int n, int bytes_pad, T* const* rx,
                                    uint64_t* const* rx_bar, int kind, uint32_t rank, uint32_t N,
                                    int lane) {
  for (uint32_t r = 0, s = 1; s < N; ++r, s <<= 1) {
    dsmem_push(buf, rx[r], rx_bar[r], bytes_pad, (rank + s) % N, lane);
    __syncwarp();
    mbar_wait(rx_bar[r], 0);
    const T* in = rx[r];
    if (kind == kSoftmaxMerge) {
      const int B = n / 2;
      for (int i = lane; i < B; i += 32) {
        const float ma = Elem<T>::to_f(buf[i]), la = Elem<T>::to_f(buf[B + i]);
        const float mb = Elem<T>::to_f(in[i]), lb = Elem<T>::to_f(in[B + i]);
        const float m = fmaxf(ma, mb);
        const float fa = (ma == -INFINITY) ? 0.f : expf(ma - m);
        const float fb = (mb == -INFINITY) ? 0.f : expf(mb - m);
        buf[i] = Elem<T>::from_f(m);
        buf[B + i] = Elem<T>::from_f(la * fa + lb * fb);
      }
    } else {
      for (int i = lane; i < n; i += 32) {
        const float a = Elem<T>::to_f(buf[i]), b = Elem<T>::to_f(in[i]);
        buf[i] = Elem<T>::from_f(kind == kMax ? fmaxf(a, b) : a + b);
      }
    }
    __syncwarp();
  }
}

// In-place all-gather: `gbuf` holds N segments of `seg_bytes` (multiple of
// 16), the local one in segment 0.  rx_bar[r] completes round r's bytes.
__device__ __forceinline__ void warp_cluster_gather(char* gbuf, int seg_bytes,
                                                    uint64_t* const* rx_bar, uint32_t rank,
                                                    uint32_t N, int lane) {
  for (uint32_t r = 0, s = 1; s < N; ++r, s <<= 1) {
    dsmem_push(gbuf, gbuf + s * seg_bytes, rx_bar[r], s * seg_bytes, (rank + s) % N, lane);
    __syncwarp();
    mbar_wait(rx_bar[r], 0);
    __syncwarp();
  }
}

}  // namespace cfb
