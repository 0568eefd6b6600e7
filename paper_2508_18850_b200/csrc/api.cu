// extern "C" surface of libcfb.so (declared in include/cfb.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "common.h"

namespace cfb {
static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
int tuned_spw() { return kMaxSlotsPerWarpHost; }
int tuned_sleep() { return 32; }

int configure_kernel(const void* fn, int max_dyn_smem, bool nonportable_cluster) {
  int dev = 0;
  CFB_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, fn})) return CFB_OK;
  CFB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem));
  if (nonportable_cluster)
    CFB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done.insert({dev, fn});
  return CFB_OK;
}
}  // namespace cfb

extern "C" {

int cfb_mha_decode(const cfb_mha_args* args, void* stream) {
  return cfb::mha_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_mla_decode(const cfb_mla_args* args, void* stream) {
  return cfb::mla_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_mla_engine_decode(const cfb_mla_engine_args* args, void* stream) {
  return cfb::mla_engine_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_splithead_decode(const cfb_splithead_args* args, void* stream) {
  return cfb::splithead_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_ffn_decode(const cfb_ffn_args* args, void* stream) {
  return cfb::ffn_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_moe_decode(const cfb_moe_args* args, void* stream) {
  return cfb::moe_decode(args, static_cast<cudaStream_t>(stream));
}

int cfb_lm_head_argmax(const cfb_lm_args* args, void* stream) {
  return cfb::lm_head_argmax(args, static_cast<cudaStream_t>(stream));
}

int cfb_embed(int dtype, const void* table, const int* tokens, float* out, int batch, int hidden,
              void* stream) {
  return cfb::embed(dtype, table, tokens, out, batch, hidden, static_cast<cudaStream_t>(stream));
}

int cfb_cluster_collective(int dtype, int op, int cluster, int n, const void* in, void* out,
                           unsigned long long* traffic, void* stream) {
  return cfb::cluster_collective(dtype, op, cluster, n, in, out, traffic,
                                 static_cast<cudaStream_t>(stream));
}

int cfb_collective_bench(int op, int channel, int cluster, int bytes, int reps, int validate,
                         const void* in, void* out, void* scratch, unsigned long long* ctr,
                         unsigned long long* ns_out, void* stream) {
  return cfb::collective_bench(op, channel, cluster, bytes, reps, validate, in, out, scratch, ctr, ns_out,
                               static_cast<cudaStream_t>(stream));
}

const char* cfb_last_error(void) { return cfb::g_err; }

const char* cfb_version(void) { return "cfb 0.1.0 sm_100a"; }

int cfb_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

}  // extern "C"
