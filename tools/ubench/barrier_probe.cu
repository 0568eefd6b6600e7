// Grid-barrier latency probe for the persistent engines: G CTAs (one per SM)
// alternate "consume K ring items" and a grid barrier, while the producer
// warp keeps streaming a large buffer through the 192 KB TMA-bulk ring (as in
// llama_step_kernel), or with the ring idle.  Thread 0 stamps globaltimer
// around every barrier; the mean over CTAs and barriers is printed per
// variant:
//   0  red.release.gpu arrival, relaxed polling, one ld.acquire (engine)
//   1  __threadfence() + relaxed red arrival, relaxed polling + ld.acquire
//   2  relaxed arrival and polling, no fence at all (NOT a valid barrier:
//      the lower bound without any memory ordering)
//   3  atom.add.acq_rel arrival (round trip), relaxed polling + ld.acquire
//   4  as 0, but only every 4th CTA arrives and polls (G/4 arrivals: the
//      global part of a hierarchical cluster-then-grid barrier)
//   5  as 0, then every CTA loads a 4096-float vector written by all CTAs
//      before the barrier (barrier + the dependent data round trip)
//   6  data-carried epochs: each CTA stores its 4096/G slice as u64 words
//      (value | epoch << 32, st.relaxed), every CTA loads all 4096 words
//      (ld.relaxed) and re-reads the stale ones until every epoch is current
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2508_18850_b200/csrc tools/ubench/barrier_probe.cu -o tools/ubench/barrier_probe
#include <cstdio>

#include "gemv.cuh"

using namespace cfb;

__device__ __forceinline__ void arrive_variant(unsigned long long* c, int v) {
  if (v == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  } else if (v == 1) {
    __threadfence();
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  } else if (v == 2) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  } else {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
  }
}

__global__ void __launch_bounds__(kThreads, 1) probe(const char* src, size_t per_cta, int items_per_round,
                                                     int rounds, int variant, int stream,
                                                     unsigned long long* counter, unsigned long long* out,
                                                     float* sink, float* vec, unsigned long long* words) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes(3));
  const Ring ring{smem, bars, bars + kNumSlots, 3, 32};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, G = gridDim.x;
  if (tid == 0) {
    ring_init(ring);
    fence_mbar_init();
  }
  __syncthreads();
  const int n_items = stream ? items_per_round * rounds * kNumConsumerWarps : 0;
  const Phase P = make_phase(src + per_cta * blockIdx.x, nullptr, n_items, kSlotBytes);
  const int per = variant == 4 ? G / 4 : G;  // arrivals per barrier
  const bool part = variant != 4 || (blockIdx.x % 4 == 0 && blockIdx.x / 4 < per);
  unsigned long long target = (ld_acquire_u64(counter) / per) * per;
  __syncthreads();
  if (warp == kNumConsumerWarps) {
    const Phase ph[1] = {P};
    produce_all(ph, ring, lane, policy_evict_first());
    return;
  }
  int cnt = 0;
  float acc = 0.f;
  unsigned long long tot = 0;
  for (int r = 0; r < rounds; ++r) {
    if (stream) {  // this warp's items of the round
      for (int j = 0; j < items_per_round; ++j) {
        const int sl = warp * ring.spw + (cnt % ring.spw);
        mbar_wait(&ring.full[sl], (cnt / ring.spw) & 1);
        acc += reinterpret_cast<const float*>(ring.slot(sl))[lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[sl]);
        ++cnt;
      }
    }
    consumer_sync();
    constexpr int kV = 4096;
    if (variant == 5 || variant == 6) {
      const int c0 = (int)((long long)blockIdx.x * kV / G), c1 = (int)((long long)(blockIdx.x + 1) * kV / G);
      unsigned long long t0 = 0;
      if (tid == 0) t0 = globaltimer();
      const unsigned ep = (unsigned)(r + 1) + 1000u * (unsigned)blockIdx.x * 0u;
      if (variant == 5) {
        for (int c = c0 + tid; c < c1; c += kConsumerThreads) vec[c] = (float)(r + c);
        consumer_sync();
        if (tid == 0) {
          target += G;
          arrive_variant(counter, 0);
          spin_until_geq(counter, target);
        }
        consumer_sync();
        float a = 0.f;
        for (int c = tid; c < kV; c += kConsumerThreads) a += __ldcg(vec + c);
        acc += a;
      } else {
        for (int c = c0 + tid; c < c1; c += kConsumerThreads) {
          const unsigned long long w = (unsigned long long)__float_as_uint((float)(r + c)) |
                                       ((unsigned long long)ep << 32);
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(words + c), "l"(w) : "memory");
        }
        float a = 0.f;
        for (int c = tid; c < kV; c += kConsumerThreads) {
          unsigned long long w;
          do {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(words + c) : "memory");
          } while ((unsigned)(w >> 32) < ep);
          a += __uint_as_float((unsigned)w);
        }
        acc += a;
      }
      consumer_sync();
      if (tid == 0) tot += globaltimer() - t0;
    } else if (tid == 0 && part) {
      const unsigned long long t0 = globaltimer();
      target += per;
      arrive_variant(counter, variant == 4 ? 0 : variant);
      spin_until_geq(counter, target);
      tot += globaltimer() - t0;
    }
    consumer_sync();
  }
  if (tid == 0) out[blockIdx.x] = tot;
  if (acc == 1234.5f) *sink = acc;
}

int main() {
  const size_t total = 4ull << 30;
  char* buf;
  unsigned long long *counter, *out;
  float* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&counter, 8);
  cudaMalloc(&out, 256 * 8);
  cudaMalloc(&sink, 4);
  float* vec;
  unsigned long long* words;
  cudaMalloc(&vec, 4096 * 4);
  cudaMalloc(&words, 4096 * 8);
  cudaMemset(words, 0, 4096 * 8);
  cudaMemset(buf, 1, total);
  cudaMemset(counter, 0, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = ring_bytes(3) + 2 * kNumSlots * 8 + 1024 * 16;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 200;
  printf("{\"sms\": %d, \"rounds\": %d, \"runs\": [\n", sms, rounds);
  bool first = true;
  unsigned long long host[256];
  for (int stream : {0, 1})
    for (int ipr : {1, 4, 16})
      for (int variant : {0, 1, 2, 3, 4, 5, 6}) {
        if (!stream && ipr > 1) continue;
        const int G = sms;
        const size_t per = (total / G) / kSlotBytes * kSlotBytes;
        if ((size_t)ipr * rounds * kNumConsumerWarps * kSlotBytes > per) continue;
        cudaMemset(words, 0, 4096 * 8);  // epochs restart at 1 every launch
        for (int rep = 0; rep < 2; ++rep)
          probe<<<G, kThreads, smem>>>(buf, per, ipr, rounds, variant, stream, counter, out, sink, vec, words);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<G, kThreads, smem>>>(buf, per, ipr, rounds, variant, stream, counter, out, sink, vec, words);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(host, out, G * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        int np = 0;
        for (int i = 0; i < G; ++i)
          if (variant != 4 || i % 4 == 0) { s += host[i]; ++np; }
        printf("%s {\"stream\": %d, \"kb_per_cta_round\": %d, \"variant\": %d, \"barrier_us\": %.3f, "
               "\"kernel_us_per_round\": %.3f}",
               first ? "" : ",\n", stream, stream ? ipr * 64 : 0, variant, s / np / rounds / 1e3,
               ms * 1e3 / rounds);
        first = false;
      }
  printf("\n]}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
