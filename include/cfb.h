/*
 * cfb.h — C ABI of libcfb.so, the B200 (sm_100a) ClusterFusion decode-step library.
 *
 * Plain pointers and sizes only; no torch types.  All device pointers are
 * caller-owned CUDA device memory; `stream` is a cudaStream_t passed as void*.
 * Every entry point is stream-ordered, allocates nothing on the hot path and
 * returns CFB_OK or a negative status; cfb_last_error() holds the message of
 * the calling thread's last failure.  Status codes map onto the reference's
 * exception hierarchy (pkg/src/clusterdec/errors.py:4-33), see cfb_status.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/clusterdec):
 *   cfb_mha_decode         <- dataflows.py:235-313  run_fused_mha_decode  (split_token, Alg. 3)
 *   cfb_mla_decode         <- dataflows.py:316-429  run_fused_mla_decode  (fused_mla, App. B.1)
 *   cfb_splithead_decode   <- dataflows.py:432-502  run_splithead_decode  (split_head, App. B.2)
 *   cfb_ffn_decode         <- oracle.py:112-131     ffn_reference(..., "silu") fused into one launch
 *   cfb_mla_engine_decode  <- dataflows.py:316-429 math, head-batched for the DeepSeek block
 *   cfb_moe_decode         <- no reference counterpart: DeepSeek-V2 MoE
 *                            (transformers DeepseekV2Moe semantics, oracle/deepseek_port.py)
 *   cfb_tc_gemm_b16        <- no reference counterpart: batch-16 projections on tcgen05 (north star)
 *   cfb_cluster_collective <- collectives.py:110-203 cluster_reduce / cluster_gather (DSMEM KAT kernel)
 *   cfb_collective_bench   <- fixtures/table1.csv:4-19 (Table 1): on-chip vs off-chip
 *                            ClusterReduce / ClusterGather latency harness
 *   cfb_lm_head_argmax, cfb_embed, cfb_llama_*  <- no reference counterpart (SPEC.md:298 non-goals);
 *                            the north-star decode loop around the fused modules.
 */
#ifndef CFB_H_
#define CFB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py) ------------------------------------------- */
enum cfb_status {
  CFB_OK = 0,
  CFB_ERR_DIMENSION = -1,      /* DimensionError: partitioning / kernel domain */
  CFB_ERR_CLUSTER_SIZE = -2,   /* InvalidClusterSize: N not a power of two in [1,16] */
  CFB_ERR_SHAPE = -3,          /* ShapeMismatch */
  CFB_ERR_SMEM = -4,           /* SmemOverflow: schedule needs more than 227 KB per CTA */
  CFB_ERR_CUDA = -5,           /* SimulationError: CUDA launch/runtime failure */
  CFB_ERR_ARGUMENT = -6        /* ValueError: null pointer / bad enum */
};

enum cfb_dtype { CFB_F16 = 2, CFB_F32 = 4 }; /* value = storage bytes (dims.dtype_bytes) */

/* cfb_mha_args.flags */
enum cfb_flags {
  CFB_APPEND = 1 << 0,       /* new token's K/V join rank N-1's segment (append_new_token) */
  CFB_WRITE_KV = 1 << 1,     /* also store the new K/V rows into the cache at position S+b */
  CFB_ROPE = 1 << 2,         /* rotate q and k_new (rotate-half convention) at position S+b */
  CFB_NORM = 1 << 3,         /* x = f16(rmsnorm(resid) * norm_w) instead of reading x */
  CFB_RESID = 1 << 4,        /* out = resid + sum_heads(...) (residual add in the epilogue) */
  CFB_STATS_MERGED = 1 << 5, /* stats_mode="merged": one SOFTMAX_MERGE pair reduce */
  CFB_PDL = 1 << 6,          /* programmatic dependent launch: the kernel may start while its
                                stream predecessor finishes (weights stream before the wait) */
  CFB_ONESHOT = 1 << 7,      /* latency-optimal cluster exchange (decode engine): one-round
                                all-to-all DSMEM gather, and ONE fused softmax-merge reduce of
                                fp32 (m, l, A) in place of the stats + attn_out reduces */
  CFB_PARTIAL = 1 << 8,      /* batch-16 tensor parallel, ranks > 0: residual-epilogue
                                projections write their partial sum only (the caller's
                                all-reduce adds the residual once, from rank 0) */
  CFB_DYN_POOL = 1 << 10,    /* fused FFN, batch 1: the last ~4 gate/up tiles per CTA are
                                work-stolen from a pool; barrier must then hold 2 u64 */
  CFB_TC_PAIR = 1 << 11      /* batched tcgen05 projections: CTA pairs (cluster 2) work on
                                two row-adjacent tiles over the same K-blocks and fetch each
                                activation block once, by TMA multicast (even tile counts;
                                odd ones fall back to single CTAs) */
};

/* DSMEM traffic counter slots (stage names of analysis.py:212-237) */
enum cfb_stage {
  CFB_STAGE_QKV_GATHER = 0,
  CFB_STAGE_STATS_MAX = 1,
  CFB_STAGE_STATS_SUM = 2,
  CFB_STAGE_STATS_MERGE = 3,
  CFB_STAGE_ATTN_OUT = 4,
  CFB_STAGE_Q_PROJ_GATHER = 5,
  CFB_STAGE_LATENT_GATHER = 6,
  CFB_STAGE_ABSORBED_Q_GATHER = 7,
  CFB_STAGE_DOWN_PROJ = 8,
  CFB_STAGE_SCORE_REDUCE = 9,
  CFB_STAGE_OUT_PROJ_REDUCE = 10,
  CFB_STAGE_COUNT = 11
};

/*
 * split_token fused attention module: one thread-block cluster of N CTAs
 * per head (grid = N x n_heads).  Layouts (T = fp16 or fp32 per dtype):
 *   x        [B][D]                      T     (unless CFB_NORM)
 *   resid    [B][D]                      fp32  (CFB_NORM / CFB_RESID)
 *   norm_w   [D]                         T
 *   w_qkv    [n_heads][N][3*Hp/N][D]     T     rank r's rows: q,k,v head-dim slices
 *   w_out    [n_heads][N][D/N][Hp]       T     rank r's rows r*D/N.. of (W_out[head])^T,
 *                                              each row chunk-rotated: logical 16-byte
 *                                              chunk k of slice row g stored at chunk
 *                                              (k + g) mod (Hp*T/16)
 *   k_cache, v_cache [n_heads][cache_cap][Hp] T
 *   rope_cs  [cache_cap][Hp/2][2]        fp32  (cos, sin)
 *   accum    [B][D]                      u64   cross-head sum in 64-bit fixed point
 *                                              (value * 2^32, two's complement), zero
 *                                              before first use; every CTA adds its
 *                                              O-proj columns with red.global.add, so
 *                                              the sum is order-independent (deterministic)
 *   out      [B][D]                      fp32  (nullable) out = [resid +] accum * 2^-32,
 *                                              after which accum is re-zeroed; NULL leaves
 *                                              the sum in accum for cfb_ffn_decode
 *   stats    [n_heads][2][B]             fp32  (score_max, score_sum) of rank 0
 * D must be a multiple of 8*N/(gcd) (16-byte rows); Hp (head_pad) a power of
 * two >= 8 holding head_dim logical dims (rest zero-padded by the caller).
 */
typedef struct cfb_mha_args {
  int dtype;
  int batch, hidden, n_heads, head_dim, head_pad;
  int cluster;
  int seq_len;          /* cached positions; ignored when step_pos != NULL */
  int cache_cap;
  int flags;
  const void* x;
  const float* resid;
  const void* norm_w;
  float eps;
  const void* w_qkv;
  const void* w_out;
  void* k_cache;
  void* v_cache;
  const float* rope_cs;
  const int* step_pos;  /* device int: S for this launch (graph-friendly) */
  float* out;
  unsigned long long* accum;
  float* stats;
  unsigned long long* traffic; /* [CFB_STAGE_COUNT] logical DSMEM bytes, or NULL */
  unsigned long long* trace;   /* [grid CTAs][16] %globaltimer phase stamps (profiling), or NULL */
} cfb_mha_args;

int cfb_mha_decode(const cfb_mha_args* args, void* stream);


/*
 * fused_mla latent-attention module (dataflows.py:316-429): one cluster of N
 * CTAs per head.  H = head_dim, R = kv_lora_rank, Hp/Rp power-of-two pads,
 * h = H/N, rs = R/N, rsp = pow2 >= max(rs, 16/T), D % N == 0.  Layouts (T):
 *   x       [B][D]
 *   w_q     [n_heads][N][ceil(h/4)][D*T/16][4][16/T]  row tiles of W_q[head][:, r*h..]^T
 *   w_kv    [N][ceil(rs/4)][D*T/16][4][16/T]          row tiles of W_kv[:, r*rs..]^T (shared)
 *   w_up    [n_heads][N][rs][Hp]     rows j of W_up[head][:, r*rs + j]^T, chunk-rotated
 *   w_down  [n_heads][N][Hp][rsp]    rows j of W_down[head][r*rs.., j]^T, chunk-rotated
 *   w_out   [n_heads][N][D/N][Hp]    as cfb_mha_args.w_out
 *   cache   [seq_len][Rp]            latent rows (shared by all heads)
 *   accum / out / stats / traffic as cfb_mha_args; flags: CFB_APPEND,
 *   CFB_STATS_MERGED, CFB_PDL, CFB_NORM (x = f16(rmsnorm(resid) * norm_w),
 *   resid [B][D] fp32, norm_w [D] T; x unused).  Batch <= 4.
 * "Chunk-rotated": logical 16-byte chunk k of row g stored at (k + g) mod nch.
 */
typedef struct cfb_mla_args {
  int dtype;
  int batch, hidden, n_heads, head_dim, head_pad, kv_rank, rank_pad;
  int cluster, seq_len, flags;
  const void* x;
  const void* w_q;
  const void* w_kv;
  const void* w_up;
  const void* w_down;
  const void* w_out;
  const void* cache;
  float* out;
  unsigned long long* accum;
  float* stats;
  unsigned long long* traffic;
  const float* resid;
  const void* norm_w;
  float eps;
} cfb_mla_args;
int cfb_mla_decode(const cfb_mla_args* args, void* stream);

/*
 * Head-batched MLA for the DeepSeek block engine (batch 1, 1..16 heads - a
 * tensor-parallel rank passes its head shard; the MMA pads to 16 - kv_lora_rank
 * 512, head_dim <= 128): same math as cfb_mla_decode (absorbed form, new latent
 * row attended once) but every weight and cache row crosses HBM once -
 * three PDL-chained launches: projections (W_q | W_kv, then W_up), split-KV
 * attention over the S+1 latent rows with tensor-core MMAs (all heads per
 * cache tile), merge + W_down + W_out into `accum` (fixed point, plain stores:
 * the block's attention head sum for cfb_moe_decode's accum_in).
 * Input x = f16(rmsnorm(resid) * norm_w).  Layouts (fp16):
 *   w_a   row tiles of [W_q^T (n_heads*H rows) ; W_kv^T (512 rows)] x D
 *   w_up  rows h*512 + j = W_up[h][:, j] (H), chunk-rotated by row index
 *   w_dn  W_down as given: [n_heads][512][H] (row h*512 + j = W_down[h][j, :])
 *   w_o   row tiles of W_out^T: row d = [W_out[0][:, d] ; ... ; W_out[15][:, d]]
 *   cache [seq_len][512]
 * Workspaces: qc [16*H + 512] fp16, qlat [16][512] fp16, part [min(SMs,
 * max_parts)][32 + 16*512] fp32, o_acc [16*H] u64 (zero: the attention launch
 * re-zeroes it every step), barrier two u64 (zero, then monotonic).
 */
typedef struct cfb_mla_engine_args {
  int hidden, n_heads, head_dim, kv_rank, seq_len, flags, max_parts;
  float eps;
  const float* resid;
  const void* norm_w;
  const void* w_a;
  const void* w_up;
  const void* w_dn;
  const void* w_o;
  const void* cache;
  void* qc;
  void* qlat;
  float* part;
  unsigned long long* o_acc;
  unsigned long long* accum;
  unsigned long long* barrier;
  unsigned long long* trace; /* nullable: [grid][16] %globaltimer stamps per CTA (profiling) */
} cfb_mla_engine_args;
int cfb_mla_engine_decode(const cfb_mla_engine_args* args, void* stream);

/*
 * split_head attention module (dataflows.py:432-502): one cluster of N CTAs
 * per head, head-dim partition throughout; reduce payloads B x (S+B) scores
 * and B x D projections (CFB_ERR_SMEM when they exceed shared memory).
 * Reference layouts (T): x [B][D], w_qkv [n_heads][D][3H], w_out
 * [n_heads][H][D], k/v_cache [n_heads][S][H].  accum/out/stats/traffic as
 * cfb_mha_args; flags: CFB_APPEND.
 */
typedef struct cfb_splithead_args {
  int dtype;
  int batch, hidden, n_heads, head_dim, cluster, seq_len, flags;
  const void* x;
  const void* w_qkv;
  const void* w_out;
  const void* k_cache;
  const void* v_cache;
  float* out;
  unsigned long long* accum;
  float* stats;
  unsigned long long* traffic;
} cfb_splithead_args;
int cfb_splithead_decode(const cfb_splithead_args* args, void* stream);

/*
 * Fused SwiGLU FFN (one launch, persistent grid, one CTA per SM):
 *   out = [r +] (silu(h w1^T) * (h w2^T)) w3^T,  h = x or f16(rmsnorm(r) * norm_w),
 *   r = resid [+ accum * 2^-32]  (accum: the attention module's fixed-point head
 *   sum, nullable; re-zeroed by this kernel).  out may alias resid.
 *   w_gu  [F][2][D]  T   row 2f = w1[f] (gate), row 2f+1 = w2[f] (up)
 *   w_dn  [D][F]     T   = w3
 *   act   [B][F]     T   workspace;  barrier: one u64 (two with CFB_DYN_POOL), zero
 *                           before first use, then monotonic (keep the same grid)
 */
typedef struct cfb_ffn_args {
  int dtype, batch, hidden, inter, flags, grid; /* grid <= 0: one CTA per SM */
  float eps;
  const void* x;
  const float* resid;
  unsigned long long* accum;
  const void* norm_w;
  const void* w_gu;
  const void* w_dn;
  void* act;
  float* out;
  unsigned long long* barrier;
  unsigned long long* trace;   /* [grid CTAs][8] %globaltimer phase stamps (profiling), or NULL */
} cfb_ffn_args;
int cfb_ffn_decode(const cfb_ffn_args* args, void* stream);

/*
 * Fused DeepSeek-V2 MoE (one launch, persistent grid, one CTA per SM):
 *   h = x or f16(rmsnorm(r) * norm_w), r = resid [+ accum_in * 2^-32]
 *   p = softmax(h W_r^T); top_k experts by p (ties: lower id), w = p * routed_scale
 *   y = sum_k w_k down_k(f16(silu(gate_k h) * up_k h)) + shared(h)
 *   out = [r +] y          (CFB_RESID; out may alias resid; accum_in re-zeroed;
 *                           CFB_PARTIAL: out = y, the tensor-parallel rank > 0 form)
 * fp16 only, batch <= 4, n_experts <= 256, top_k <= 16, hidden a multiple of 8
 * up to 512 or one of 1024/2048/4096.  Layouts (fp16), Q = max(1, hidden/512):
 *   w_router [E][D]
 *   w_gu     [E][inter/2][D/8][4][8]   row tiles (gate 2t, gate 2t+1, up 2t, up 2t+1)
 *   w_dn     [E][inter/8][Q][8][D/Q]   blocks of W_down^T: 8 intermediate rows x D/Q
 *   s_gu / s_dn: shared experts (width shared_inter = n_shared * inter), same layouts
 *   accum    [B][D] u64 workspace, zero before first use (re-zeroed)
 *   barrier  two u64 (grid barrier, route counter), zero before first use; both are
 *            monotonic, so a workspace must always be used with the same grid
 *   logits   [B][E] fp32 workspace: router logits of the last launch
 *   route_idx/route_w [B][top_k] (nullable): selected experts / gate weights
 */
typedef struct cfb_moe_args {
  int dtype, batch, hidden, n_experts, top_k, inter, shared_inter, flags, grid;
  float eps, routed_scale;
  const void* x;
  const float* resid;
  unsigned long long* accum_in;
  const void* norm_w;
  const void* w_router;
  const void* w_gu;
  const void* w_dn;
  const void* s_gu;
  const void* s_dn;
  float* part;                 /* [grid][batch*hidden] fp32 workspace: per-CTA MoE partial sums */
  float* out;
  int* route_idx;
  float* route_w;
  unsigned long long* barrier;
  float* logits;
  unsigned long long* trace;   /* [grid CTAs][16] %globaltimer phase stamps (profiling), or NULL */
} cfb_moe_args;
int cfb_moe_decode(const cfb_moe_args* args, void* stream);

/* Final RMSNorm + LM head + greedy argmax (first index of the max, numpy
 * semantics).  w [V][D] T; logits [B][V] fp32 (nullable); cand_* [grid][B]
 * workspace; ticket one u32 (zero); token_out [B]; step_pos (nullable) is
 * incremented once the token is written. */
typedef struct cfb_lm_args {
  int dtype, batch, hidden, vocab, grid, flags; /* flags: CFB_PDL */
  float eps;
  const float* resid;
  const void* norm_w;
  const void* w;
  float* logits;
  float* cand_val;
  int* cand_idx;
  unsigned* ticket;
  int* token_out;
  int* step_pos;
} cfb_lm_args;
int cfb_lm_head_argmax(const cfb_lm_args* args, void* stream);

/*
 * Batch-16 projection on the tcgen05 tensor cores (swap-AB: weights = MMA M,
 * batch = N = 16; TMEM accumulators): y[n][m] = sum_k W[m][k] x[n][k].
 *   w_packed  W (M x K fp16) in UMMA blocks: [M/128][K/64][k-step 4][K half 2]
 *             [row group 16][8 rows][8]  (K-major, no swizzle; see csrc/tc_gemm.cu)
 *   x         [16][K] fp16 row-major; x_packed: 16*K fp16 workspace
 *   y_acc     [16][M] u64 fixed-point workspace, zero before first use
 *   y         [16][M] fp32 out (= [resid +] y_acc * 2^-32, y_acc re-zeroed), or NULL
 *             to leave the sum in y_acc.   M % 128 == 0, K % 64 == 0.
 */
int cfb_tc_gemm_b16(const void* w_packed, const void* x, void* x_packed, unsigned long long* y_acc,
                    float* y, const float* resid, int M, int K, int flags, void* stream);

/*
 * Batch-16 SwiGLU FFN block on tcgen05: resid[n] += FFN(f16(rmsnorm(resid[n]) * norm_w))
 * for 16 rows: RMSNorm+pack -> [w1; w2] projection -> SiLU*mul+pack -> w3
 * projection -> residual add (3 PDL-chained launches; the last CTA to finish
 * a 128-row tile applies SiLU*mul / the residual add).  w_gu = pack of the
 * gate/up rows interleaved per 64: [w1[0:64]; w2[0:64]; w1[64:128]; ...]
 * (2F x D), w_dn = pack of w3 (D x F) (cfb_tc_gemm_b16 layout).
 * Workspaces: xp 16*D fp16, gu_acc 16*2F u64 (zero), ap 16*F fp16, out_acc
 * 16*D u64 (zero), ticket (2F + D)/128 ints (zero).  hidden % 128 == 0,
 * inter % 64 == 0.
 */
typedef struct cfb_ffn_b16_args {
  int hidden, inter, flags;
  float eps;
  float* resid;
  const void* norm_w;
  const void* w_gu;
  const void* w_dn;
  void* xp;
  unsigned long long* gu_acc;
  void* ap;
  unsigned long long* out_acc;
  int* ticket;
  int batch;  /* rows = MMA N: 16 (or 0) or 32; the workspaces above scale with it */
  float* slots; /* cfb_b16_slots_floats(hidden, 0, inter, batch) floats: per-contributor partial tiles */
} cfb_ffn_b16_args;
/* Floats of the partial-slot workspace (`slots`) the batched projections need:
 * per 128-row tile, one fp32 [batch][128] partial per contributing CTA, summed
 * in CTA order by the tile's finishing CTA (deterministic, no atomics). */
size_t cfb_b16_slots_floats(int hidden, int n_heads, int inter, int batch);
int cfb_ffn_b16(const cfb_ffn_b16_args* args, void* stream);

/*
 * One Llama decoder layer for 16 INDEPENDENT sequences (own KV caches and
 * positions), batch>1 path on tcgen05: RMSNorm+pack -> QKV projection whose
 * finishing epilogue applies RoPE at pos[n] and appends k, v to sequence n's
 * cache -> split-KV attention over rows 0..pos[n] -> O projection + residual
 * -> batch-16 FFN block.  resid [16][hidden] fp32 is updated in place.
 *   w_qkv  packed [q heads ; k heads ; v heads] x 128 rows (3*hidden x hidden)
 *   w_o    packed W_out^T (hidden x hidden); w_gu / w_dn as cfb_ffn_b16
 *   k_cache, v_cache [16][n_heads][cache_cap][128] fp16; rope_cs [cap][64][2]
 *   pos [16] device ints: the new token's position per sequence (not advanced;
 *   cfb_b16_advance adds 1 to all of them)
 * Workspaces (zeroed once): xp 16*max(hidden, inter) fp16, q16 16*hidden fp16,
 * qkv_acc 16*3*hidden u64, part 16*n_heads*ceil(max_len/128)*130 fp32,
 * o_acc 16*hidden u64, gu_acc 16*2*inter u64, ap 16*inter fp16,
 * ticket (3*n_heads*128 + 2*hidden + 2*inter)/128 + 16*n_heads ints (zero).
 * flags: CFB_PDL, CFB_PARTIAL.
 */
typedef struct cfb_b16_layer_args {
  int hidden, n_heads, inter, cache_cap, max_len, flags;
  /* stage: 0 whole layer, 1 attention half only, 2 FFN half only (tensor parallel:
   * one all-reduce of resid after each half; n_heads / inter are then the rank's
   * shard: n_heads*128 <= hidden, inter % 64 == 0) */
  int stage;
  float eps;
  float* resid;
  const void* attn_norm;
  const void* ffn_norm;
  const void* w_qkv;
  const void* w_o;
  const void* w_gu;
  const void* w_dn;
  void* k_cache;
  void* v_cache;
  const float* rope_cs;
  const int* pos;
  void* xp;
  void* q16;
  unsigned long long* qkv_acc;
  float* part;
  unsigned long long* o_acc;
  unsigned long long* gu_acc;
  void* ap;
  int* ticket;
  /* paged KV cache (NULL = the contiguous layout above): block_table [16][max_pages]
   * page ids; k_cache / v_cache are then page pools [n_pages][n_heads][128][128]
   * fp16 (page = CFB_KV_PAGE positions of all heads); position p of sequence n
   * lives in page block_table[n][p / CFB_KV_PAGE] at row p % CFB_KV_PAGE */
  const int* block_table;
  int max_pages;
  /* sequences = MMA N: 16 (or 0) or 32.  Every "16" above is this batch
   * (caches, pos, table rows, workspaces); a sequence with pos -1 is inactive */
  int batch;
  float* slots; /* cfb_b16_slots_floats(hidden, n_heads, inter, batch) floats */
} cfb_b16_layer_args;
#define CFB_KV_PAGE 128
int cfb_llama_b16_layer(const cfb_b16_layer_args* args, void* stream);
int cfb_b16_advance(int* pos, int batch, void* stream); /* batch 0 = 16; pos -1 stays -1 */
/* KV writer (prefill / import): rows [start, start + count) of sequence seq
 * from k_src / v_src [n_heads][count][128] fp16 (device) into the paged pools
 * (block_table as above; the pages must already be assigned) or, with
 * block_table NULL, into the contiguous [16][n_heads][cache_cap][128] caches. */
int cfb_b16_kv_write(void* k_cache, void* v_cache, const int* block_table, int max_pages, int cache_cap,
                     int n_heads, int seq, int start, int count, const void* k_src, const void* v_src,
                     void* stream);
/* Batch-16 final RMSNorm + LM head (tcgen05, w_lm packed V x hidden) + greedy
 * argmax per sequence (first index of the max): tokens [16]; logits [16][V]
 * fp32 or NULL; xp 16*hidden fp16, y_acc 16*V u64 (zero) and scratch
 * CFB_B16_ARGMAX_SCRATCH u64 (zero) workspaces.  vocab % 128 == 0.  Then
 * cfb_embed(batch 16) gathers the next inputs. */
#define CFB_B16_ARGMAX_SCRATCH (65 * 32)
int cfb_b16_lm_head(const float* resid, const void* norm_w, const void* w_lm, int vocab, int hidden,
                    float eps, void* xp, unsigned long long* y_acc, int* tokens, float* logits,
                    unsigned long long* scratch, int batch, void* stream); /* batch 0 = 16, or 32 */

/* out[b][:] = float(table[tokens[b]][:]) */
int cfb_embed(int dtype, const void* table, const int* tokens, float* out, int batch, int hidden,
              void* stream);

/*
 * Whole-model greedy decode step (Llama2 family, batch 1):
 *   embed -> n_layers x (split_token attention module [norm, rope, kv append,
 *   fixed-point head sum] -> fused FFN [residual + head sum, norm, residual])
 *   -> final norm + LM head + argmax, every launch with CFB_PDL.
 * Per-layer weight pointers are in the layouts above; rope_cs [cache_cap][H/2][2].
 * The engine owns its small workspace; the CUDA graph of one step advances
 * the device-side position, so replays decode consecutive tokens.
 */
enum cfb_engine_kind {
  CFB_ENGINE_LAYERED = 0,    /* one launch per block half: split_token cluster kernel (DSMEM
                                exchange) + fused FFN kernel, PDL-chained (2L+2 launches) */
  CFB_ENGINE_PERSISTENT = 1, /* ONE persistent launch per step (csrc/decode_step.cu): the
                                producer warps stream every layer's weights without stopping;
                                the attention module of a head runs on one N-CTA cluster
                                (split_token, DSMEM gather/exchange), grid barriers between
                                block halves; head_dim 128 */
  CFB_ENGINE_PERSISTENT_FLAT = 2, /* as PERSISTENT, but the attention is split over all SMs
                                and its partials are exchanged through global memory with
                                per-head flags (a different partitioning, kept as an A/B) */
  CFB_ENGINE_PERSISTENT_NODSMEM = 3 /* as PERSISTENT (same clusters, same partitioning), but
                                the ClusterGather and the (m, l, A) exchange go through global
                                memory: the paper's "without DSMEM" ablation */
};
typedef struct cfb_llama_config {
  int dtype, n_layers, hidden, n_heads, head_dim, inter, vocab, cache_cap, cluster;
  float eps;
  int engine; /* cfb_engine_kind */
} cfb_llama_config;
typedef struct cfb_llama_weights {
  const void* embed;
  const void* final_norm;
  const void* lm_head;
  const float* rope_cs;
  const void* const* attn_norm;
  const void* const* w_qkv;
  const void* const* w_out;
  const void* const* ffn_norm;
  const void* const* w_gu;
  const void* const* w_dn;
  void* const* k_cache;
  void* const* v_cache;
} cfb_llama_weights;
typedef struct cfb_llama cfb_llama;
int cfb_llama_create(const cfb_llama_config* cfg, const cfb_llama_weights* w, cfb_llama** out);
int cfb_llama_destroy(cfb_llama* m);
int cfb_llama_set_state(cfb_llama* m, int pos, int token, void* stream);
int cfb_llama_step(cfb_llama* m, void* stream);
int cfb_llama_capture(cfb_llama* m, void* stream);
int cfb_llama_replay(cfb_llama* m, void* stream);
int cfb_llama_buffers(cfb_llama* m, float** logits, int** token, int** pos, float** resid);
int cfb_llama_launches_per_step(const cfb_llama* m);
/* stream-ordered copies between the engine and host memory (either may be NULL) */
int cfb_llama_read(cfb_llama* m, int* token_host, float* logits_host, void* stream);

/*
 * Tensor parallelism (north-star (d)): each rank's engine is created with its
 * shard - n_heads / size heads (W_qkv, W_out, KV cache of those heads), inter /
 * size FFN columns (gate/up rows, down columns), vocab / size LM-head rows
 * starting at vocab_offset - and is driven part by part so the caller can put
 * one all-reduce after each block half:
 *   EMBED; per layer: ATTN -> allreduce(accum, int64 SUM: the fixed-point head
 *   sum, exact) -> FFN (rank 0 adds the residual, other ranks write their
 *   partial) -> allreduce(resid, fp32 SUM); HEAD (local argmax packed into
 *   argkey) -> allreduce(argkey, int64 MAX) -> TP_TOKEN (global token, pos++).
 * With size 1 the parts are exactly cfb_llama_step.
 */
enum cfb_engine_part {
  CFB_PART_EMBED = 0,
  CFB_PART_ATTN = 1,
  CFB_PART_FFN = 2,
  CFB_PART_HEAD = 3,
  CFB_PART_TP_TOKEN = 4
};
/* accum [D] u64, resid [D] fp32, argkey one u64: caller-owned, zeroed buffers the
 * engine then uses instead of its own (so a communicator can address them), or NULL */
int cfb_llama_set_tp(cfb_llama* m, int rank, int size, int vocab_offset, unsigned long long* accum,
                     float* resid, unsigned long long* argkey);
int cfb_llama_enqueue(cfb_llama* m, int part, int layer, void* stream);
/* Fused tensor parallel (persistent engines only): the step kernel itself does
 * both all-reduces of every layer and the vocabulary-shard argmax, pushing
 * 64-bit fixed-point partial sums straight into every rank's exchange block over
 * NVLink peer memory and meeting the other ranks at a cross-rank counter; one
 * launch per token, no NCCL call.  xch_peers [size]: each rank's exchange
 * block (cfb_tp_xch_bytes(hidden), zeroed) as addressable from THIS device -
 * cfb_ipc_open'ed for remote ranks, the locally allocated one for `rank`.
 * emulated != 0: all ranks share this GPU (tests): a plain launch on `grid`
 * CTAs per rank, sized by the caller so every rank is resident.  timeout_ns > 0
 * bounds each cross-rank wait (cfb_llama_check then reports 2). */
int cfb_llama_set_tp_fused(cfb_llama* m, int rank, int size, int vocab_offset, void* const* xch_peers,
                           int emulated, int grid, long long timeout_ns);
size_t cfb_tp_xch_bytes(int hidden);
/* NVLS (NVLink SHARP multicast) for the fused all-reduce (SURVEY 8(e) next
 * step): uc_sum / mc_sum are the unicast and multicast mappings of this rank's
 * copy of a multicast buffer of >= cfb_tp_nvls_bytes(hidden) bytes (zeroed).
 * The step kernel then adds each sum slice ONCE with multimem.red.add.u64 on
 * mc_sum (the switch updates every rank's copy) instead of once per peer, and
 * reads / re-zeroes uc_sum; barriers and the argmax stay on the exchange
 * blocks.  NULL, NULL = the peer-memory pushes.  Call after
 * cfb_llama_set_tp_fused. */
int cfb_llama_set_tp_nvls(cfb_llama* m, void* uc_sum, void* mc_sum);
size_t cfb_tp_nvls_bytes(int hidden);
/* Multicast objects (one physical copy per member GPU; nvls.cu):
 * creator: cfb_nvls_create(bytes, ndev) [+ cfb_nvls_export_fd]; other members:
 * cfb_nvls_import_fd(creator pid, fd, bytes, ndev) (pidfd_getfd); then every
 * member cfb_nvls_add_device (all of them before any bind) and
 * cfb_nvls_bind(device) -> unicast / multicast mappings of its zeroed copy.
 * An emulated group on one GPU: ndev 1, the ranks share the mappings. */
typedef struct cfb_nvls cfb_nvls;
int cfb_nvls_supported(int device, int* supported);
int cfb_nvls_create(size_t bytes, int ndev, cfb_nvls** out);
int cfb_nvls_export_fd(cfb_nvls* h, int* fd);
int cfb_nvls_import_fd(int pid, int fd, size_t bytes, int ndev, cfb_nvls** out);
int cfb_nvls_add_device(cfb_nvls* h, int device);
int cfb_nvls_bind(cfb_nvls* h, int device, void** uc, void** mc);
size_t cfb_nvls_size(const cfb_nvls* h);
int cfb_nvls_destroy(cfb_nvls* h);
/* Engine options (set before cfb_llama_capture; a captured graph keeps the
 * values it was captured with). */
enum cfb_llama_option {
  CFB_OPT_L2_PREFETCH = 1, /* persistent engines: bytes per CTA of the next phase, past what
                             the smem ring holds, prefetched into L2 at each grid barrier
                             (HBM keeps streaming while the CTA waits); 0 = off */
  CFB_OPT_PLAIN_LAUNCH = 2, /* persistent engines: 1 = launch without the cooperative
                             attribute (the grid is sized co-resident either way; for
                             profilers that cannot replay cooperative cluster launches) */
  CFB_OPT_RING_SLOTS = 3,   /* persistent engines: 8 KB ring slots per consumer warp
                             (1..3: 64 / 128 / 192 KB per CTA); 0 = the deepest that fits */
  CFB_OPT_POOL_TILES = 4    /* persistent engines: gate/up tiles per CTA handed out
                             dynamically at the end of the phase (work stealing); 0 = 4 */
};
int cfb_llama_set_option(cfb_llama* m, int option, long long value);
/* Inter-process peer memory for the exchange blocks: cudaMalloc + zero + IPC
 * handle (64 bytes) / open a peer's handle (lazy peer access) / close / free. */
int cfb_ipc_alloc(size_t bytes, void** dev, void* handle);
int cfb_ipc_open(const void* handle, void** dev);
int cfb_ipc_close(void* dev);
int cfb_dev_free(void* dev);
int cfb_llama_tp_buffers(cfb_llama* m, unsigned long long** accum, float** resid,
                         unsigned long long** argkey);
int cfb_llama_write_token(cfb_llama* m, const int* token_host, void* stream);
/* Persistent engine only: per-CTA globaltimer stamps [n_layers][grid][8] (phase
 * boundaries of csrc/decode_step.cu) written each step into `trace` (device, or
 * NULL to stop); returns the grid size through *grid. */
int cfb_llama_set_trace(cfb_llama* m, unsigned long long* trace, int* grid);
/* Persistent cluster engines (PERSISTENT / PERSISTENT_NODSMEM) only: paged KV
 * cache (SURVEY §8(f) rank 4 at batch 1).  k_cache / v_cache of the weights
 * are then per-layer page pools of 128-position pages: row r of head h sits at
 * element h * head_stride + block_table[r / 128] * page_stride + (r % 128) *
 * head_dim.  Page-major pools [n_pages][n_heads][128][head_dim] (the batched
 * path's layout: page_stride = n_heads * 128 * head_dim, head_stride = 128 *
 * head_dim) and head-major pools [n_heads][n_pages][128][head_dim]
 * (page_stride = 128 * head_dim, head_stride = n_pages * 128 * head_dim) are
 * both expressible.  `block_table` [max_pages] (device, int32, -1 = not
 * reserved), max_pages * 128 >= cache_cap.  A step whose new row lands on an
 * unreserved page does nothing and reports err 1 (cfb_llama_check).  NULL
 * returns to the contiguous caches.  Set before cfb_llama_capture (a captured
 * graph keeps the table pointer; the table's CONTENTS may change between
 * replays). */
int cfb_llama_set_kv_pages(cfb_llama* m, const int* block_table, int max_pages, long long page_stride,
                           long long head_stride);
/* Device-side status of the last steps: *err_host = 1 if a step found pos + 1 >
 * cache_cap and did nothing, 2 if a fused tensor-parallel step gave up waiting
 * for its peers (stream-ordered read, then the flag is cleared). */
int cfb_llama_check(cfb_llama* m, int* err_host, void* stream);

/* One ClusterReduce (op 0=sum,1=max,2=softmax_merge) or ClusterGather (op 3)
 * over N CTAs of one cluster; in/out [N][n] T.  Test kernel for the DSMEM
 * primitives (reference KATs). */
int cfb_cluster_collective(int dtype, int op, int cluster, int n, const void* in, void* out,
                           unsigned long long* traffic, void* stream);

/* Table-1 latency harness (fixtures/table1.csv:4-19): one
 * cluster of N CTAs runs `reps` ClusterReduce (op 0, fp16 sum of `bytes` per
 * rank) or ClusterGather (op 3, bytes/N per rank) collectives on operands in
 * shared memory, over DSMEM bulk copies (channel 0) or through global memory /
 * L2 (channel 1).  validate = 1: operands from in [N][bytes] fp16, results to
 * out [N][bytes]; validate = 0 (timing): synthetic operands, results folded
 * into a checksum.  scratch (1 MB) and ctr (one u64, zeroed) for channel 1.
 * *ns_out (device) = mean ns per collective on rank 0. */
int cfb_collective_bench(int op, int channel, int cluster, int bytes, int reps, int validate,
                         const void* in, void* out, void* scratch, unsigned long long* ctr,
                         unsigned long long* ns_out, void* stream);

const char* cfb_last_error(void);
const char* cfb_version(void);
int cfb_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CFB_H_ */
