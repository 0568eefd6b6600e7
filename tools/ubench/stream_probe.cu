// Streaming-bandwidth probe for the cfb ring engine (csrc/stream.cuh): G CTAs
// (one per SM) each stream a contiguous share of a 4 GiB buffer through the
// TMA-bulk ring (spw slots of 8 KB per consumer warp) with a trivial
// consumer.  Answers: how many SMs does it take to saturate HBM, and what
// per-SM bandwidth does a given ring depth sustain?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2508_18850_b200/csrc tools/ubench/stream_probe.cu -o /tmp/stream_probe
#include <cstdio>
#include <vector>

#include "gemv.cuh"

using namespace cfb;

// mode 0: touch one word per lane per slot; mode 1: the engine's tile GEMV
// (4-row tiles of K = 4096 fp16, FHFMA, activations fp16 in smem)
__global__ void __launch_bounds__(kThreads, 1) probe(const char* src, size_t per_cta, int spw, int* sink,
                                                     int mode) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes(3));
  const Ring ring{smem, bars, bars + kNumSlots, spw, 32};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr int K = 4096;
  const Phase P = mode == 0
      ? make_phase(src + per_cta * blockIdx.x, nullptr, (int)(per_cta / kSlotBytes), kSlotBytes)
      : make_phase(src + per_cta * blockIdx.x, nullptr, (int)(per_cta / (4 * K * 2)), 4 * K * 2, true);
  __half* xs = reinterpret_cast<__half*>(smem + ring_bytes(3) + 2 * kNumSlots * 8);
  for (int i = tid; i < K; i += kThreads) xs[i] = __float2half(0.001f * (i % 7));
  __syncthreads();
  if (warp == kNumConsumerWarps) {
    const Phase ph[1] = {P};
    produce_all(ph, ring, lane, policy_evict_last());
    return;
  }
  int cnt = 0, acc = 0;
  float facc = 0.f;
  consume_phase(P, ring, warp, lane, cnt, [&](const Item& it, const char* slot) {
    if (mode == 0) {
      acc += reinterpret_cast<const int*>(slot)[lane * 64];
    } else {
      tile_item<__half, 1, true>(P, it, slot, xs, K, 1, lane,
                                 [&](int row, const float (&s)[1]) { facc += s[0]; });
    }
  });
  if (facc == 1234.5f) acc = 1;
  if (acc == 0x12345678) *sink = acc;
}

int main() {
  const size_t total = 4ull << 30;
  char* buf;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = ring_bytes(3) + 2 * kNumSlots * 8 + 1024 * 20;  // force 1 CTA/SM
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"runs\": [\n", sms);
  bool first = true;
  for (size_t span : {total, (size_t)64 << 20})  // HBM stream, then an L2-resident 64 MiB
  for (int mode : {0, 1})
  for (int spw : {2, 3}) {
    for (int G : {32, 64, 96, 128, 132, 148}) {
      if (G > sms) continue;
      const size_t per = (span / G) / (4 * 4096 * 2) * (4 * 4096 * 2);
      for (int r = 0; r < 2; ++r) probe<<<G, kThreads, smem>>>(buf, per, spw, sink, mode);
      cudaEventRecord(e0);
      const int reps = span == total ? 5 : 100;
      for (int r = 0; r < reps; ++r) probe<<<G, kThreads, smem>>>(buf, per, spw, sink, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = (double)per * G * reps / (ms * 1e-3) / 1e9;
      printf("%s {\"span_mb\": %zu, \"mode\": %d, \"spw\": %d, \"ring_kb\": %d, \"grid\": %d, \"gbs\": %.1f, \"gbs_per_sm\": %.1f}", first ? "" : ",\n",
             span >> 20, mode, spw, spw * 64, G, gbs, gbs / G);
      first = false;
    }
  }
  printf("\n]}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
