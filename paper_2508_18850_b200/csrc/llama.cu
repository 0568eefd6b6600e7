// Whole-model greedy decode engine (Llama2 family, batch 1): the native
// runtime around the fused kernels.  One step = embed -> n_layers x
// (split_token attention module, fused SwiGLU FFN) -> LM head + argmax; the
// step is captured once into a CUDA graph and replayed, and the device-side
// position/token it advances make consecutive replays decode consecutive
// tokens without any host work.
#include <cstring>
#include <vector>

#include "common.h"
#include "ptx.cuh"

struct cfb_llama {
  cfb_llama_config cfg;
  std::vector<const void*> attn_norm, w_qkv, w_out, ffn_norm, w_gu, w_dn;
  std::vector<void*> k_cache, v_cache;
  const void* embed = nullptr;
  const void* final_norm = nullptr;
  const void* lm_head = nullptr;
  const float* rope_cs = nullptr;
  // workspace (engine-owned)
  float* resid = nullptr;             // fp32 residual stream [D]
  unsigned long long* accum = nullptr; // attention head sum, fixed point [D]
  void* act = nullptr;
  unsigned long long* barrier = nullptr;
  float* logits = nullptr;
  float* cand_val = nullptr;
  int* cand_idx = nullptr;
  unsigned* lm_ticket = nullptr;
  int* token = nullptr;
  int* pos = nullptr;
  unsigned long long* argkey = nullptr;  // TP: packed (logit, -index) of the local argmax
  int tp_rank = 0, tp_size = 1, vocab_offset = 0;
  int ext = 0;  // bit mask: accum / resid / argkey are caller-owned
  // persistent engine (csrc/decode_step.cu)
  void** dev_ptrs = nullptr;            // 8 x n_layers per-layer pointers, device copy
  void* pqkv = nullptr;                 // q|k|v rows of the current layer
  float* partials = nullptr;            // attention partials [nh][grid][132]
  unsigned long long* pbarrier = nullptr;
  unsigned long long* counters = nullptr;  // [2 nh] flat per-head flags + [sms] per-cluster
  int* err = nullptr;
  unsigned long long* trace = nullptr;
  int grid = 0;
  // fused tensor parallel (persistent engine, in-kernel all-reduce over peer memory)
  int tp_fused = 0, emulated = 0;
  int l2_prefetch = 0;  // CFB_OPT_L2_PREFETCH
  int plain_launch = 0; // CFB_OPT_PLAIN_LAUNCH
  int ring_spw = 0;     // CFB_OPT_RING_SLOTS
  int pool_per_cta = 0; // CFB_OPT_POOL_TILES
  const int* kv_pages = nullptr;  // cfb_llama_set_kv_pages: block table, or null (contiguous)
  long long kv_pstride = 0, kv_hstride = 0;
  long long timeout_ns = 0;
  unsigned long long** xch_dev = nullptr;  // [tp_size] exchange blocks as this device sees them
  float* resid2 = nullptr;
  unsigned long long* uc_sum = nullptr;  // NVLS sums (cfb_llama_set_tp_nvls) or null
  unsigned long long* mc_sum = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

namespace {

int alloc_zero(void** p, size_t bytes) {
  CFB_CUDA(cudaMalloc(p, bytes));
  CFB_CUDA(cudaMemset(*p, 0, bytes));
  return CFB_OK;
}

// Tensor-parallel argmax: order-preserving 32-bit key of the local maximum
// logit in the high word, 0xffffffff - global index in the low word, so an
// int64 MAX all-reduce yields the largest logit and, among equal logits, the
// smallest index (numpy argmax semantics across vocabulary shards).
__global__ void tp_argmax_pack_kernel(const float* logits, const int* token, int vocab_offset,
                                      unsigned long long* key) {
  cfb::pdl_wait();
  const int t = *token;
  const unsigned u = __float_as_uint(logits[t]);
  const unsigned ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // unsigned-monotone
  // high word flipped to signed order: NCCL's int64 MAX compares signed
  *key = ((unsigned long long)(ord ^ 0x80000000u) << 32) | (0xffffffffu - (unsigned)(t + vocab_offset));
}
__global__ void tp_argmax_unpack_kernel(const unsigned long long* key, int* token, int* pos) {
  *token = (int)(0xffffffffu - (unsigned)(*key & 0xffffffffull));
  *pos += 1;
}

int enqueue_embed(cfb_llama* m, cudaStream_t st) {
  return cfb::embed(m->cfg.dtype, m->embed, m->token, m->resid, 1, m->cfg.hidden, st, true);
}

int enqueue_attn(cfb_llama* m, int l, cudaStream_t st) {
  const cfb_llama_config& c = m->cfg;
  cfb_mha_args a = {};
  a.dtype = c.dtype;
  a.batch = 1;
  a.hidden = c.hidden;
  a.n_heads = c.n_heads;
  a.head_dim = c.head_dim;
  a.head_pad = c.head_dim;
  a.cluster = c.cluster;
  a.cache_cap = c.cache_cap;
  a.flags = CFB_APPEND | CFB_WRITE_KV | CFB_ROPE | CFB_ONESHOT | CFB_PDL | CFB_NORM;
  a.resid = m->resid;
  a.norm_w = m->attn_norm[l];
  a.eps = c.eps;
  a.w_qkv = m->w_qkv[l];
  a.w_out = m->w_out[l];
  a.k_cache = m->k_cache[l];
  a.v_cache = m->v_cache[l];
  a.rope_cs = m->rope_cs;
  a.step_pos = m->pos;
  a.out = nullptr;  // the head sum stays in accum for the FFN prologue (TP: all-reduced first)
  a.accum = m->accum;
  return cfb::mha_decode(&a, st);
}

int enqueue_ffn(cfb_llama* m, int l, cudaStream_t st) {
  const cfb_llama_config& c = m->cfg;
  cfb_ffn_args f = {};
  f.dtype = c.dtype;
  f.batch = 1;
  f.hidden = c.hidden;
  f.inter = c.inter;
  // TP: only rank 0 adds the residual, so the all-reduce of resid counts it once;
  // the last gate/up tiles are work-stolen (CFB_DYN_POOL)
  f.flags = CFB_NORM | CFB_PDL | CFB_DYN_POOL | (m->tp_rank == 0 ? CFB_RESID : 0);
  f.eps = c.eps;
  f.resid = m->resid;
  f.accum = m->accum;
  f.norm_w = m->ffn_norm[l];
  f.w_gu = m->w_gu[l];
  f.w_dn = m->w_dn[l];
  f.act = m->act;
  f.out = m->resid;
  f.barrier = m->barrier;
  return cfb::ffn_decode(&f, st);
}

int enqueue_head(cfb_llama* m, cudaStream_t st) {
  const cfb_llama_config& c = m->cfg;
  cfb_lm_args h = {};
  h.dtype = c.dtype;
  h.batch = 1;
  h.hidden = c.hidden;
  h.vocab = c.vocab;
  h.eps = c.eps;
  h.flags = CFB_PDL;
  h.resid = m->resid;
  h.norm_w = m->final_norm;
  h.w = m->lm_head;
  h.logits = m->logits;
  h.cand_val = m->cand_val;
  h.cand_idx = m->cand_idx;
  h.ticket = m->lm_ticket;
  h.token_out = m->token;
  h.step_pos = m->tp_size > 1 ? nullptr : m->pos;  // TP: advanced after the global argmax
  int rc = cfb::lm_head_argmax(&h, st);
  if (rc || m->tp_size == 1) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1);
  cfg.stream = st;
  cfb::LaunchAttrs at(0, true);
  cfg.attrs = at.a;
  cfg.numAttrs = at.n;
  CFB_CUDA(cudaLaunchKernelEx(&cfg, tp_argmax_pack_kernel, (const float*)m->logits,
                              (const int*)m->token, m->vocab_offset, m->argkey));
  return CFB_OK;
}

int enqueue_tp_token(cfb_llama* m, cudaStream_t st) {
  tp_argmax_unpack_kernel<<<1, 1, 0, st>>>(m->argkey, m->token, m->pos);
  CFB_CUDA(cudaGetLastError());
  return CFB_OK;
}

int enqueue_part(cfb_llama* m, int part, int layer, cudaStream_t st) {
  switch (part) {
    case CFB_PART_EMBED: return enqueue_embed(m, st);
    case CFB_PART_ATTN: return enqueue_attn(m, layer, st);
    case CFB_PART_FFN: return enqueue_ffn(m, layer, st);
    case CFB_PART_HEAD: return enqueue_head(m, st);
    case CFB_PART_TP_TOKEN: return enqueue_tp_token(m, st);
  }
  return cfb::set_error(CFB_ERR_ARGUMENT, "unknown engine part %d", part);
}

int enqueue_persistent(cfb_llama* m, cudaStream_t st) {
  const cfb_llama_config& c = m->cfg;
  const int L = c.n_layers;
  cfb::LlamaStepArgs a = {};
  a.n_layers = L;
  a.hidden = c.hidden;
  a.n_heads = c.n_heads;
  a.head_dim = c.head_dim;
  a.inter = c.inter;
  a.vocab = c.vocab;
  a.cache_cap = c.cache_cap;
  a.cluster = c.cluster;
  a.grid = m->grid;
  a.cluster_attn = c.engine == CFB_ENGINE_PERSISTENT ? 1 : c.engine == CFB_ENGINE_PERSISTENT_NODSMEM ? 2 : 0;
  a.eps = c.eps;
  void** d = m->dev_ptrs;
  a.attn_norm = d;
  a.w_qkv = d + L;
  a.w_out = d + 2 * L;
  a.ffn_norm = d + 3 * L;
  a.w_gu = d + 4 * L;
  a.w_dn = d + 5 * L;
  a.k_cache = d + 6 * L;
  a.v_cache = d + 7 * L;
  a.kv_pages = m->kv_pages;
  a.kv_pstride = m->kv_pstride;
  a.kv_hstride = m->kv_hstride;
  a.embed = m->embed;
  a.final_norm = m->final_norm;
  a.lm_head = m->lm_head;
  a.rope_cs = m->rope_cs;
  a.resid = m->resid;
  a.accA = m->accum;
  a.act = m->act;
  a.qkv = m->pqkv;
  a.partials = m->partials;
  a.barrier = m->pbarrier;
  a.counters = m->counters;
  a.pool_ctr = m->pbarrier + 1;
  a.logits = m->logits;
  a.cand_val = m->cand_val;
  a.cand_idx = m->cand_idx;
  a.ticket = m->lm_ticket;
  a.token = m->token;
  a.pos = m->pos;
  a.err = m->err;
  a.trace = m->trace;
  a.l2_prefetch = m->l2_prefetch;
  a.ring_spw = m->ring_spw;
  a.pool_per_cta = m->pool_per_cta;
  a.emulated = m->plain_launch;
  if (m->tp_fused) {
    a.tp_size = m->tp_size;
    a.tp_rank = m->tp_rank;
    a.vocab_offset = m->vocab_offset;
    a.emulated = m->emulated || m->plain_launch;
    a.xch = m->xch_dev;
    a.resid2 = m->resid2;
    a.uc_sum = m->uc_sum;
    a.mc_sum = m->mc_sum;
    a.timeout_ns = m->timeout_ns;
  }
  return cfb::llama_step_launch(&a, st);
}

int enqueue_step(cfb_llama* m, cudaStream_t st) {
  if (m->tp_size > 1 && !m->tp_fused)
    return cfb::set_error(CFB_ERR_ARGUMENT,
                          "tensor-parallel engines are driven part by part (collectives between)");
  if (m->cfg.engine != CFB_ENGINE_LAYERED) return enqueue_persistent(m, st);
  int rc = enqueue_embed(m, st);
  for (int l = 0; !rc && l < m->cfg.n_layers; ++l)
    if (!(rc = enqueue_attn(m, l, st))) rc = enqueue_ffn(m, l, st);
  return rc ? rc : enqueue_head(m, st);
}

}  // namespace

extern "C" {

int cfb_llama_create(const cfb_llama_config* cfg, const cfb_llama_weights* w, cfb_llama** out) {
  using cfb::set_error;
  if (!cfg || !w || !out) return set_error(CFB_ERR_ARGUMENT, "null argument");
  if (cfg->n_layers < 1 || !w->attn_norm || !w->w_qkv || !w->w_out || !w->ffn_norm || !w->w_gu ||
      !w->w_dn || !w->k_cache || !w->v_cache || !w->embed || !w->final_norm || !w->lm_head ||
      !w->rope_cs)
    return set_error(CFB_ERR_ARGUMENT, "missing weight pointers");
  cfb_llama* m = new cfb_llama();
  m->cfg = *cfg;
  const int L = cfg->n_layers;
  m->attn_norm.assign(w->attn_norm, w->attn_norm + L);
  m->w_qkv.assign(w->w_qkv, w->w_qkv + L);
  m->w_out.assign(w->w_out, w->w_out + L);
  m->ffn_norm.assign(w->ffn_norm, w->ffn_norm + L);
  m->w_gu.assign(w->w_gu, w->w_gu + L);
  m->w_dn.assign(w->w_dn, w->w_dn + L);
  m->k_cache.assign(w->k_cache, w->k_cache + L);
  m->v_cache.assign(w->v_cache, w->v_cache + L);
  m->embed = w->embed;
  m->final_norm = w->final_norm;
  m->lm_head = w->lm_head;
  m->rope_cs = w->rope_cs;
  const size_t D = cfg->hidden;
  int rc = 0;
  int sms = cfb_device_sm_count();
  if (sms <= 0) sms = 148;
  if ((rc = alloc_zero((void**)&m->resid, D * 4)) || (rc = alloc_zero((void**)&m->accum, D * 8)) ||
      (rc = alloc_zero(&m->act, (size_t)cfg->inter * cfg->dtype)) ||
      (rc = alloc_zero((void**)&m->barrier, 16)) ||
      (rc = alloc_zero((void**)&m->logits, (size_t)cfg->vocab * 4)) ||
      (rc = alloc_zero((void**)&m->cand_val, (size_t)sms * 4)) ||
      (rc = alloc_zero((void**)&m->cand_idx, (size_t)sms * 4)) ||
      (rc = alloc_zero((void**)&m->lm_ticket, 4)) || (rc = alloc_zero((void**)&m->token, 4)) ||
      (rc = alloc_zero((void**)&m->pos, 4)) || (rc = alloc_zero((void**)&m->argkey, 8))) {
    cfb_llama_destroy(m);
    return rc;
  }
  if (cfg->engine != CFB_ENGINE_LAYERED) {
    if (cfg->engine != CFB_ENGINE_PERSISTENT && cfg->engine != CFB_ENGINE_PERSISTENT_FLAT &&
        cfg->engine != CFB_ENGINE_PERSISTENT_NODSMEM) {
      cfb_llama_destroy(m);
      return set_error(CFB_ERR_ARGUMENT, "unknown engine kind %d", cfg->engine);
    }
    if (cfg->dtype != CFB_F16 || cfg->head_dim != 128) {
      cfb_llama_destroy(m);
      return set_error(CFB_ERR_DIMENSION, "persistent engine: fp16, head_dim 128");
    }
    cfb::LlamaStepArgs ga = {};
    ga.n_layers = L;
    ga.hidden = cfg->hidden;
    ga.n_heads = cfg->n_heads;
    ga.head_dim = cfg->head_dim;
    ga.inter = cfg->inter;
    ga.vocab = cfg->vocab;
    ga.cache_cap = cfg->cache_cap;
    ga.cluster = cfg->cluster;
    ga.cluster_attn = cfg->engine == CFB_ENGINE_PERSISTENT ? 1 : cfg->engine == CFB_ENGINE_PERSISTENT_NODSMEM ? 2 : 0;
    if ((rc = cfb::llama_step_grid(&ga, &m->grid, nullptr, nullptr))) {
      cfb_llama_destroy(m);
      return rc;
    }
    const int N = cfg->cluster;
    const size_t qkv_rows = (size_t)cfg->n_heads * N * ((3 * cfg->head_dim / N + 3) / 4) * 4;
    std::vector<const void*> host(8 * (size_t)L);
    for (int l = 0; l < L; ++l) {
      host[l] = w->attn_norm[l];
      host[L + l] = w->w_qkv[l];
      host[2 * L + l] = w->w_out[l];
      host[3 * L + l] = w->ffn_norm[l];
      host[4 * L + l] = w->w_gu[l];
      host[5 * L + l] = w->w_dn[l];
      host[6 * L + l] = w->k_cache[l];
      host[7 * L + l] = w->v_cache[l];
    }
    if ((rc = alloc_zero((void**)&m->dev_ptrs, host.size() * sizeof(void*))) ||
        (rc = alloc_zero(&m->pqkv, qkv_rows * 2)) ||
        (rc = alloc_zero((void**)&m->partials, (size_t)cfg->n_heads * sms * 132 * 4)) ||

        (rc = alloc_zero((void**)&m->pbarrier, 8 * (1 + (size_t)L))) ||
        (rc = alloc_zero((void**)&m->counters, ((size_t)2 * cfg->n_heads + sms) * 8)) ||
        (rc = alloc_zero((void**)&m->err, 4))) {
      cfb_llama_destroy(m);
      return rc;
    }
    const cudaError_t e = cudaMemcpy(m->dev_ptrs, host.data(), host.size() * sizeof(void*),
                                     cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cfb_llama_destroy(m);
      return set_error(CFB_ERR_CUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
    }
  }
  *out = m;
  return CFB_OK;
}

int cfb_llama_destroy(cfb_llama* m) {
  if (!m) return CFB_OK;
  if (m->exec) cudaGraphExecDestroy(m->exec);
  if (m->graph) cudaGraphDestroy(m->graph);
  void* bufs[] = {(m->ext & 2) ? nullptr : m->resid, (m->ext & 1) ? nullptr : m->accum,
                  m->act, m->barrier, m->logits, m->cand_val, m->cand_idx, m->lm_ticket, m->token,
                  m->pos, (m->ext & 4) ? nullptr : m->argkey, m->dev_ptrs, m->pqkv,
                  m->partials, m->pbarrier, m->counters, m->err, m->xch_dev, m->resid2};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete m;
  return CFB_OK;
}

int cfb_llama_set_state(cfb_llama* m, int pos, int token, void* stream) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (pos < 0 || pos >= m->cfg.cache_cap)
    return cfb::set_error(CFB_ERR_DIMENSION, "pos %d outside cache capacity %d", pos, m->cfg.cache_cap);
  // tensor parallel: the local vocabulary is a shard, the token is global
  if (token < 0 || token >= m->cfg.vocab * m->tp_size)
    return cfb::set_error(CFB_ERR_DIMENSION, "token out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static thread_local int host[2];
  host[0] = pos;
  host[1] = token;
  CFB_CUDA(cudaMemcpyAsync(m->pos, &host[0], 4, cudaMemcpyHostToDevice, st));
  CFB_CUDA(cudaMemcpyAsync(m->token, &host[1], 4, cudaMemcpyHostToDevice, st));
  CFB_CUDA(cudaStreamSynchronize(st));
  return CFB_OK;
}

int cfb_llama_step(cfb_llama* m, void* stream) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  return enqueue_step(m, static_cast<cudaStream_t>(stream));
}

int cfb_llama_capture(cfb_llama* m, void* stream) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m->exec) {
    cudaGraphExecDestroy(m->exec);
    m->exec = nullptr;
  }
  if (m->graph) {
    cudaGraphDestroy(m->graph);
    m->graph = nullptr;
  }
  CFB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int rc = enqueue_step(m, st);
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CFB_CUDA(e);
  m->graph = g;
  CFB_CUDA(cudaGraphInstantiate(&m->exec, g, 0));
  return CFB_OK;
}

int cfb_llama_replay(cfb_llama* m, void* stream) {
  if (!m || !m->exec) return cfb::set_error(CFB_ERR_ARGUMENT, "engine has no captured graph");
  CFB_CUDA(cudaGraphLaunch(m->exec, static_cast<cudaStream_t>(stream)));
  return CFB_OK;
}

int cfb_llama_buffers(cfb_llama* m, float** logits, int** token, int** pos, float** resid) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (logits) *logits = m->logits;
  if (token) *token = m->token;
  if (pos) *pos = m->pos;
  if (resid) *resid = m->resid;
  return CFB_OK;
}

int cfb_llama_launches_per_step(const cfb_llama* m) {
  if (m && m->cfg.engine != CFB_ENGINE_LAYERED && (m->tp_size == 1 || m->tp_fused)) return 1;
  return m ? 2 + 2 * m->cfg.n_layers + (m->tp_size > 1 ? 2 : 0) : 0;
}

int cfb_llama_set_tp(cfb_llama* m, int rank, int size, int vocab_offset, unsigned long long* accum,
                     float* resid, unsigned long long* argkey) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (size < 1 || rank < 0 || rank >= size || vocab_offset < 0)
    return cfb::set_error(CFB_ERR_ARGUMENT, "bad tensor-parallel rank %d / size %d", rank, size);
  m->tp_rank = rank;
  m->tp_size = size;
  m->vocab_offset = vocab_offset;
  // caller-owned (e.g. torch-allocated, so a communicator can address them) buffers
  // replace the engine's own; they must be zero-initialised like the originals
  if (accum) {
    cudaFree(m->accum);
    m->accum = accum;
    m->ext |= 1;
  }
  if (resid) {
    cudaFree(m->resid);
    m->resid = resid;
    m->ext |= 2;
  }
  if (argkey) {
    cudaFree(m->argkey);
    m->argkey = argkey;
    m->ext |= 4;
  }
  return CFB_OK;
}

int cfb_llama_set_tp_fused(cfb_llama* m, int rank, int size, int vocab_offset, void* const* xch_peers,
                           int emulated, int grid, long long timeout_ns) {
  using cfb::set_error;
  if (!m || !xch_peers) return set_error(CFB_ERR_ARGUMENT, "null argument");
  if (m->cfg.engine == CFB_ENGINE_LAYERED)
    return set_error(CFB_ERR_ARGUMENT, "fused tensor parallel needs a persistent engine");
  if (size < 2 || size > 64 || rank < 0 || rank >= size || vocab_offset < 0)
    return set_error(CFB_ERR_ARGUMENT, "bad tensor-parallel rank %d / size %d", rank, size);
  for (int t = 0; t < size; ++t)
    if (!xch_peers[t]) return set_error(CFB_ERR_ARGUMENT, "missing exchange block of rank %d", t);
  if (grid > 0) {  // emulated ranks on one GPU: each gets a share of the SMs
    cfb::LlamaStepArgs ga = {};
    ga.n_layers = m->cfg.n_layers;
    ga.hidden = m->cfg.hidden;
    ga.n_heads = m->cfg.n_heads;
    ga.head_dim = m->cfg.head_dim;
    ga.inter = m->cfg.inter;
    ga.vocab = m->cfg.vocab;
    ga.cache_cap = m->cfg.cache_cap;
    ga.cluster = m->cfg.cluster;
    ga.grid = grid;
    ga.cluster_attn = m->cfg.engine == CFB_ENGINE_PERSISTENT ? 1 : m->cfg.engine == CFB_ENGINE_PERSISTENT_NODSMEM ? 2 : 0;
    if (const int rc = cfb::llama_step_grid(&ga, &m->grid, nullptr, nullptr)) return rc;
    if (m->grid > grid) return set_error(CFB_ERR_ARGUMENT, "grid %d does not fit %d", grid, m->grid);
  }
  if (!m->xch_dev) CFB_CUDA(cudaMalloc((void**)&m->xch_dev, 64 * sizeof(void*)));
  CFB_CUDA(cudaMemcpy(m->xch_dev, xch_peers, (size_t)size * sizeof(void*), cudaMemcpyHostToDevice));
  if (!m->resid2) {
    CFB_CUDA(cudaMalloc((void**)&m->resid2, (size_t)m->cfg.hidden * 4));
    CFB_CUDA(cudaMemset(m->resid2, 0, (size_t)m->cfg.hidden * 4));
  }
  m->tp_rank = rank;
  m->tp_size = size;
  m->vocab_offset = vocab_offset;
  m->tp_fused = 1;
  m->emulated = emulated ? 1 : 0;
  m->timeout_ns = timeout_ns;
  return CFB_OK;
}

size_t cfb_tp_xch_bytes(int hidden) { return cfb::tp_xch_bytes(hidden); }

size_t cfb_tp_nvls_bytes(int hidden) { return (size_t)6 * hidden * sizeof(unsigned long long); }

int cfb_llama_set_tp_nvls(cfb_llama* m, void* uc_sum, void* mc_sum) {
  using cfb::set_error;
  if (!m) return set_error(CFB_ERR_ARGUMENT, "null engine");
  if (!m->tp_fused) return set_error(CFB_ERR_ARGUMENT, "NVLS sums need cfb_llama_set_tp_fused first");
  if ((uc_sum == nullptr) != (mc_sum == nullptr)) return set_error(CFB_ERR_ARGUMENT, "uc_sum and mc_sum go together");
  m->uc_sum = static_cast<unsigned long long*>(uc_sum);
  m->mc_sum = static_cast<unsigned long long*>(mc_sum);
  return CFB_OK;
}

int cfb_llama_set_option(cfb_llama* m, int option, long long value) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  switch (option) {
    case CFB_OPT_L2_PREFETCH:
      if (value < 0 || value > (64 << 20) || value % 16)
        return cfb::set_error(CFB_ERR_ARGUMENT, "l2 prefetch bytes must be a multiple of 16 in [0, 64 MB]");
      m->l2_prefetch = (int)value;
      return CFB_OK;
    case CFB_OPT_PLAIN_LAUNCH:
      m->plain_launch = value ? 1 : 0;
      return CFB_OK;
    case CFB_OPT_POOL_TILES:
      if (value < 0 || value > 64) return cfb::set_error(CFB_ERR_ARGUMENT, "pool tiles per CTA must be in [0, 64]");
      m->pool_per_cta = (int)value;
      return CFB_OK;
    case CFB_OPT_RING_SLOTS:
      if (value < 0 || value > 3)
        return cfb::set_error(CFB_ERR_ARGUMENT, "ring slots per consumer warp must be in [0, 3]");
      m->ring_spw = (int)value;
      return CFB_OK;
  }
  return cfb::set_error(CFB_ERR_ARGUMENT, "unknown engine option %d", option);
}

int cfb_ipc_alloc(size_t bytes, void** dev, void* handle) {
  if (!dev || !handle || !bytes) return cfb::set_error(CFB_ERR_ARGUMENT, "null argument");
  CFB_CUDA(cudaMalloc(dev, bytes));
  CFB_CUDA(cudaMemset(*dev, 0, bytes));
  CFB_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), *dev));
  return CFB_OK;
}

int cfb_ipc_open(const void* handle, void** dev) {
  if (!dev || !handle) return cfb::set_error(CFB_ERR_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CFB_CUDA(cudaIpcOpenMemHandle(dev, h, cudaIpcMemLazyEnablePeerAccess));
  return CFB_OK;
}

int cfb_ipc_close(void* dev) {
  if (dev) CFB_CUDA(cudaIpcCloseMemHandle(dev));
  return CFB_OK;
}

int cfb_dev_free(void* dev) {
  if (dev) CFB_CUDA(cudaFree(dev));
  return CFB_OK;
}

int cfb_llama_enqueue(cfb_llama* m, int part, int layer, void* stream) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if ((part == CFB_PART_ATTN || part == CFB_PART_FFN) && (layer < 0 || layer >= m->cfg.n_layers))
    return cfb::set_error(CFB_ERR_ARGUMENT, "layer %d out of range", layer);
  return enqueue_part(m, part, layer, static_cast<cudaStream_t>(stream));
}

int cfb_llama_tp_buffers(cfb_llama* m, unsigned long long** accum, float** resid,
                         unsigned long long** argkey) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (accum) *accum = m->accum;
  if (resid) *resid = m->resid;
  if (argkey) *argkey = m->argkey;
  return CFB_OK;
}

int cfb_llama_read(cfb_llama* m, int* token_host, float* logits_host, void* stream) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (token_host) CFB_CUDA(cudaMemcpyAsync(token_host, m->token, 4, cudaMemcpyDeviceToHost, st));
  if (logits_host)
    CFB_CUDA(cudaMemcpyAsync(logits_host, m->logits, (size_t)m->cfg.vocab * 4, cudaMemcpyDeviceToHost, st));
  return CFB_OK;
}

int cfb_llama_write_token(cfb_llama* m, const int* token_host, void* stream) {
  if (!m || !token_host) return cfb::set_error(CFB_ERR_ARGUMENT, "null argument");
  CFB_CUDA(cudaMemcpyAsync(m->token, token_host, 4, cudaMemcpyHostToDevice,
                           static_cast<cudaStream_t>(stream)));
  return CFB_OK;
}

int cfb_llama_set_trace(cfb_llama* m, unsigned long long* trace, int* grid) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (m->cfg.engine == CFB_ENGINE_LAYERED)
    return cfb::set_error(CFB_ERR_ARGUMENT, "tracing needs a persistent engine");
  m->trace = trace;
  if (grid) *grid = m->grid;
  return CFB_OK;
}

int cfb_llama_set_kv_pages(cfb_llama* m, const int* block_table, int max_pages, long long page_stride,
                           long long head_stride) {
  if (!m) return cfb::set_error(CFB_ERR_ARGUMENT, "null engine");
  if (m->cfg.engine != CFB_ENGINE_PERSISTENT && m->cfg.engine != CFB_ENGINE_PERSISTENT_NODSMEM)
    return cfb::set_error(CFB_ERR_ARGUMENT, "paged KV needs a persistent cluster engine");
  if (m->cfg.head_dim != 128) return cfb::set_error(CFB_ERR_DIMENSION, "paged KV needs head_dim 128");
  if (block_table && (long long)max_pages * 128 < m->cfg.cache_cap)
    return cfb::set_error(CFB_ERR_DIMENSION, "block table of %d pages < cache_cap %d positions", max_pages,
                          m->cfg.cache_cap);
  if (block_table && (page_stride <= 0 || head_stride < 0 || page_stride % 8 || head_stride % 8))
    return cfb::set_error(CFB_ERR_ARGUMENT, "paged KV strides must be positive multiples of 8 elements");
  m->kv_pages = block_table;
  m->kv_pstride = page_stride;
  m->kv_hstride = head_stride;
  return CFB_OK;
}

int cfb_llama_check(cfb_llama* m, int* err_host, void* stream) {
  if (!m || !err_host) return cfb::set_error(CFB_ERR_ARGUMENT, "null argument");
  *err_host = 0;
  if (!m->err) return CFB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CFB_CUDA(cudaMemcpyAsync(err_host, m->err, 4, cudaMemcpyDeviceToHost, st));
  CFB_CUDA(cudaStreamSynchronize(st));
  CFB_CUDA(cudaMemsetAsync(m->err, 0, 4, st));
  return CFB_OK;
}

}  // extern "C"
