// Host-side helpers shared by the cfb translation units: error state and
// status codes of the C ABI (include/cfb.h).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstddef>

#include "../../include/cfb.h"

namespace cfb {

constexpr int kMaxSmem = 227 * 1024;
constexpr int kMaxSlotsPerWarpHost = 3;  // == kMaxSlotsPerWarp (stream.cuh)

// Launch attributes shared by the cfb kernels: optional cluster shape and
// programmatic dependent launch (the kernel may start while its predecessor
// in the stream finishes; it orders itself with griddepcontrol.wait).
struct LaunchAttrs {
  cudaLaunchAttribute a[2];
  int n = 0;
  LaunchAttrs(int cluster, bool pdl) {
    if (cluster > 0) {
      a[n].id = cudaLaunchAttributeClusterDimension;
      a[n].val.clusterDim.x = cluster;
      a[n].val.clusterDim.y = 1;
      a[n].val.clusterDim.z = 1;
      ++n;
    }
    if (pdl) {
      a[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      a[n].val.programmaticStreamSerializationAllowed = 1;
      ++n;
    }
  }
};

int set_error(int code, const char* fmt, ...);

// Ring depth (slots per consumer warp) and producer idle back-off cap (ns):
// fixed at the values the round-1 sweeps picked.
int tuned_spw();
int tuned_sleep();
// Per-(device, kernel) attribute cache: sets the dynamic shared-memory limit
// (and non-portable cluster sizes) once per device, thread-safe.
int configure_kernel(const void* fn, int max_dyn_smem, bool nonportable_cluster);

#define CFB_CUDA(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ::cfb::set_error(CFB_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,         \
                              cudaGetErrorString(e_), __FILE__, __LINE__);          \
  } while (0)

// Persistent whole-step decode kernel (csrc/decode_step.cu).  Per-layer
// pointer arrays live in DEVICE memory (the kernel walks all layers).
struct LlamaStepArgs {
  int n_layers, hidden, n_heads, head_dim, inter, vocab, cache_cap, cluster, grid;
  int cluster_attn;  // 1: attention module on DSMEM clusters; 2: same clusters, exchanges through
                     // global memory (no-DSMEM ablation); 0: flattened over all SMs, global exchange
  float eps;
  const void* const* attn_norm;
  const void* const* w_qkv;
  const void* const* w_out;
  const void* const* ffn_norm;
  const void* const* w_gu;
  const void* const* w_dn;
  void* const* k_cache;
  void* const* v_cache;
  const int* kv_pages;        // paged KV block table [cache_cap / 128] or NULL (contiguous)
  long long kv_pstride, kv_hstride;  // paged: elements between pages / between heads
  const void* embed;
  const void* final_norm;
  const void* lm_head;
  const float* rope_cs;
  float* resid;               // [D]
  unsigned long long* accA;   // [D] attention head sum (fixed point)
  void* act;                  // [F]
  void* qkv;
  float* partials;
  unsigned long long* barrier;
  unsigned long long* counters;
  unsigned long long* pool_ctr;  // [n_layers] gate/up work-stealing counters, or NULL (static)
  float* logits;
  float* cand_val;
  int* cand_idx;
  unsigned* ticket;
  int* token;
  int* pos;
  int* err;
  unsigned long long* trace;
  // tensor parallel (tp_size > 1): this rank's shard of heads / FFN columns /
  // LM-head rows; the all-reduces run inside the kernel over peer memory
  int tp_size, tp_rank, vocab_offset;
  int emulated;                  // ranks share one GPU: plain (non-cooperative) launch, grid given
  unsigned long long* const* xch;  // DEVICE array [tp_size] of the ranks' exchange blocks
                                   // (tp_xch_bytes(hidden) each, zeroed), as this device sees them
  float* resid2;                 // [D] second residual buffer (layer-parity rotation)
  unsigned long long* uc_sum;    // NVLS: this rank's copy of the [6][D] sums (or null)
  unsigned long long* mc_sum;    // NVLS: its multicast mapping (multimem.red target)
  long long timeout_ns;          // cross-rank wait bound (err = 2 on expiry), 0 = none
  int l2_prefetch;               // bytes/CTA prefetched into L2 past the ring at each barrier
  int ring_spw;                  // ring slots per consumer warp (8 KB each); 0 = the deepest that fits
  int pool_per_cta;              // work-stolen gate/up tiles per CTA; 0 = 4
};
// Exchange block of one tensor-parallel rank: reduced attention / FFN sums
// [3][D] u64 each (fixed point), the cross-rank barrier counter, the argmax
// key and the token counter (each on its own 128-byte line).
size_t tp_xch_bytes(int hidden);
int llama_step_launch(const LlamaStepArgs* a, cudaStream_t st);
int llama_step_smem(int D, int F, int nh, int N, int tpr, int V, int G, int max_spw, int* spw_out);
int llama_step_grid(const LlamaStepArgs* a, int* grid_out, int* smem_out, int* spw_out);

int mha_decode(const cfb_mha_args* a, cudaStream_t st);
int mha_finalize(float* out, const float* resid, unsigned long long* accum, int n, cudaStream_t st);
int mla_decode(const cfb_mla_args* a, cudaStream_t st);
int mla_engine_decode(const cfb_mla_engine_args* a, cudaStream_t st);
int splithead_decode(const cfb_splithead_args* a, cudaStream_t st);
int ffn_decode(const cfb_ffn_args* a, cudaStream_t st);
int ffn_b16(const cfb_ffn_b16_args* a, cudaStream_t st);
int moe_decode(const cfb_moe_args* a, cudaStream_t st);
int lm_head_argmax(const cfb_lm_args* a, cudaStream_t st);
int embed(int dtype, const void* table, const int* tokens, float* out, int B, int D,
          cudaStream_t st, bool pdl = false);
int collective_bench(int op, int channel, int N, int bytes, int reps, int validate, const void* in, void* out,
                     void* scratch, unsigned long long* ctr, unsigned long long* ns_out, cudaStream_t st);
int cluster_collective(int dtype, int op, int cluster, int n, const void* in, void* out,
                       unsigned long long* traffic, cudaStream_t st);

}  // namespace cfb
