"""Tensor-parallel Llama decode (north-star (d), BASELINE.json config #5).

One process per GPU.  Rank r of `world` holds a Megatron shard of every
layer: heads [r*nh/W, (r+1)*nh/W) (their W_qkv columns, W_out rows and KV
cache), FFN columns [r*F/W, (r+1)*F/W) (gate/up rows, down columns) and LM
head rows [r*V/W, (r+1)*V/W); embedding and norms are replicated.  A step is
the native engine driven part by part with exactly one all-reduce per block
half (NCCL over NVLink via torch.distributed, captured in the same CUDA
graph as the kernels):

    EMBED
    per layer:  ATTN  -> all_reduce(accum, int64 SUM)   attention half: the
                         64-bit fixed-point head sum - integer, so the sum over
                         ranks is exact and order-independent
                FFN   -> all_reduce(resid, fp32 SUM)    FFN half: rank 0 adds
                         the residual, the others contribute their partial
    HEAD  -> all_reduce(argkey, int64 MAX)   (logit, -index) of each shard's
             argmax: the global greedy token (first index of the max)
    TP_TOKEN

The same schedule is ``tp_step`` below, parameterised by the compute and
communication operations, so the CPU tests run it with the numpy oracle and
gloo (world size 2) and the GPU runs it with the kernels and NCCL.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import numpy as np

from . import _native
from .exceptions import DimensionError
from .llama import LlamaConfig, LlamaDecoder

PART_EMBED, PART_ATTN, PART_FFN, PART_HEAD, PART_TP_TOKEN = 0, 1, 2, 3, 4


# ------------------------------------------------------------------ sharding
def check_tp(cfg: LlamaConfig, world: int) -> None:
    if cfg.n_heads % world or cfg.inter % (8 * world) or cfg.vocab % (4 * world):
        raise DimensionError(f"tensor-parallel size {world} must divide the heads, inter/8 and vocab/4 "
                             f"({cfg.n_heads}, {cfg.inter}, {cfg.vocab})")


def local_config(cfg: LlamaConfig, world: int, cluster: int | None = None) -> LlamaConfig:
    """The per-rank model shape; `cluster` defaults to keeping ~128 CTAs per
    attention launch (4 x heads at TP1, up to 16 CTAs per head)."""
    check_tp(cfg, world)
    nh = cfg.n_heads // world
    if cluster is None:
        cluster = cfg.cluster
        while nh * cluster < 128 and cluster < 16 and cfg.head_dim % (2 * cluster) == 0:
            cluster *= 2
    # ranks are driven part by part with a collective between block halves:
    # the layered engine (the persistent step kernel has no cross-GPU exchange)
    return replace(cfg, n_heads=nh, inter=cfg.inter // world, vocab=cfg.vocab // world,
                   cluster=cluster, engine="layered")


def shard_layer(lp: dict, rank: int, world: int) -> dict:
    """Megatron shard of one logical layer (``random_llama_params`` layout)."""
    nh = lp["w_qkv"].shape[0] // world
    F = lp["w1"].shape[0] // world
    hs, fs = slice(rank * nh, (rank + 1) * nh), slice(rank * F, (rank + 1) * F)
    return dict(attn_norm=lp["attn_norm"], ffn_norm=lp["ffn_norm"], w_qkv=lp["w_qkv"][hs],
                w_out=lp["w_out"][hs], k_cache=lp["k_cache"][hs], v_cache=lp["v_cache"][hs],
                w1=lp["w1"][fs], w2=lp["w2"][fs], w3=lp["w3"][:, fs])


def shard_params(params: dict, rank: int, world: int) -> dict:
    V = params["lm_head"].shape[0] // world
    return dict(layers=[shard_layer(lp, rank, world) for lp in params["layers"]],
                embed=params["embed"], final_norm=params["final_norm"],
                lm_head=params["lm_head"][rank * V:(rank + 1) * V])


def pack_argmax_key(value: float, index: int) -> int:
    """Host twin of the device packing (csrc/llama.cu tp_argmax_pack_kernel):
    signed-int64 key whose MAX is the largest value, ties to the smallest index."""
    u = int(np.float32(value).view(np.uint32))
    ord_ = (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)
    key = ((ord_ ^ 0x80000000) << 32) | (0xFFFFFFFF - index)
    return key - (1 << 64) if key >= (1 << 63) else key


def unpack_argmax_key(key: int) -> int:
    return 0xFFFFFFFF - (key & 0xFFFFFFFF)


def tp_step(ops, n_layers: int) -> None:
    """The tensor-parallel decode schedule (one step).  `ops` supplies
    embed/attn/ffn/head/token compute and the three collectives."""
    ops.embed()
    for l in range(n_layers):
        ops.attn(l)
        ops.allreduce_heads()      # int64 SUM of the fixed-point head sum
        ops.ffn(l)
        ops.allreduce_resid()      # fp32 SUM (residual added by rank 0 only)
    ops.head()
    ops.allreduce_argmax()         # int64 MAX of the packed (logit, -index) keys
    ops.token()


# ------------------------------------------------------------------ GPU driver
class _EngineOps:
    """tp_step operations bound to a rank's native engine + NCCL group."""

    def __init__(self, dec: "TPLlamaDecoder"):
        self.d = dec

    def _enq(self, part, layer=0):
        _native.check(self.d.lib.cfb_llama_enqueue(self.d.eng._h, part, layer, self.d.sp()))

    def embed(self):
        self._enq(PART_EMBED)

    def attn(self, l):
        self._enq(PART_ATTN, l)

    def ffn(self, l):
        self._enq(PART_FFN, l)

    def head(self):
        self._enq(PART_HEAD)

    def token(self):
        if self.d.world > 1:
            self._enq(PART_TP_TOKEN)

    def _ar(self, t, op):
        if self.d.world > 1 or self.d.force_collectives:
            import torch.distributed as dist
            dist.all_reduce(t, op=op, group=self.d.group)

    def allreduce_heads(self):
        import torch.distributed as dist
        self._ar(self.d.accum, dist.ReduceOp.SUM)

    def allreduce_resid(self):
        import torch.distributed as dist
        self._ar(self.d.resid, dist.ReduceOp.SUM)

    def allreduce_argmax(self):
        import torch.distributed as dist
        if self.d.world > 1:
            self._ar(self.d.argkey, dist.ReduceOp.MAX)


class TPLlamaDecoder:
    """Rank-local tensor-parallel decoder.  `group` is a torch.distributed
    NCCL process group (None: the default group)."""

    def __init__(self, cfg: LlamaConfig, rank: int, world: int, cache_cap: int, *, params=None,
                 seed: int = 0, group=None, cluster: int | None = None,
                 force_collectives: bool = False):
        import torch
        self.cfg, self.rank, self.world, self.group = cfg, rank, world, group
        self.lcfg = local_config(cfg, world, cluster)
        self.force_collectives = force_collectives
        if params is not None:
            self.eng = LlamaDecoder.from_params(self.lcfg, shard_params(params, rank, world), cache_cap)
        else:
            self.eng = LlamaDecoder.random(self.lcfg, cache_cap, seed=seed)
        dev = self.eng.dev
        self.accum = torch.zeros(cfg.hidden, device=dev, dtype=torch.int64)
        self.resid = torch.zeros(cfg.hidden, device=dev, dtype=torch.float32)
        self.argkey = torch.zeros(1, device=dev, dtype=torch.int64)
        torch.cuda.synchronize()  # zeroed on the current stream; the engine uses its own
        self.lib = _native.lib()
        self.lib.cfb_llama_set_tp.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3
        self.lib.cfb_llama_enqueue.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        _native.check(self.lib.cfb_llama_set_tp(self.eng._h, rank, world, rank * self.lcfg.vocab,
                                                self.accum.data_ptr(), self.resid.data_ptr(),
                                                self.argkey.data_ptr()))
        self.ops = _EngineOps(self)
        self.graph = None

    @property
    def stream(self):
        return self.eng.stream

    def sp(self) -> int:
        return self.eng.stream.cuda_stream

    @property
    def launches_per_step(self) -> int:
        return 2 + 2 * self.cfg.n_layers + (2 if self.world > 1 else 0)

    def set_state(self, pos: int, token: int) -> None:
        self.eng.set_state(pos, token)

    def step(self) -> None:
        import torch
        with torch.cuda.stream(self.eng.stream):
            tp_step(self.ops, self.cfg.n_layers)

    def capture(self) -> None:
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.eng.stream):
            tp_step(self.ops, self.cfg.n_layers)

    def replay(self) -> None:
        import torch
        with torch.cuda.stream(self.eng.stream):  # stream-ordered with token()/logits reads
            self.graph.replay()

    def token(self) -> int:
        return self.eng.token()

    def logits_local(self) -> np.ndarray:
        return self.eng.logits()


# ------------------------------------------------------------------ batch 16
def shard_layer_b16(lp: dict, rank: int, world: int) -> dict:
    """Megatron shard of one logical layer for the batch-16 tcgen05 path: the
    FFN column shard is zero-padded to a multiple of 64 (a zero gate/up row
    gives silu(0) * 0 = 0, a zero down column adds nothing)."""
    sh = shard_layer(lp, rank, world)
    F = sh["w1"].shape[0]
    Fp = -(-F // 64) * 64
    if Fp != F:
        pad = Fp - F
        D = sh["w1"].shape[1]
        sh["w1"] = np.concatenate([sh["w1"], np.zeros((pad, D), np.float32)], 0)
        sh["w2"] = np.concatenate([sh["w2"], np.zeros((pad, D), np.float32)], 0)
        sh["w3"] = np.concatenate([sh["w3"], np.zeros((sh["w3"].shape[0], pad), np.float32)], 1)
    return sh


class TPBatchedLlama:
    """Rank-local shard of the batch-16 independent-sequence stack; one
    all-reduce of the residual stream per block half (rank 0 adds the
    residual, the others their partial: CFB_PARTIAL)."""

    def __init__(self, cfg: LlamaConfig, rank: int, world: int, cache_cap: int, *, params=None,
                 caches=None, seed: int = 0, group=None):
        from .batched import BatchedLlama
        if cfg.n_heads % world:
            raise DimensionError(f"tensor-parallel size {world} must divide the heads")
        self.cfg, self.rank, self.world, self.group = cfg, rank, world, group
        nh = cfg.n_heads // world
        Fp = -(-(cfg.inter // world) // 64) * 64
        self.lcfg = replace(cfg, n_heads=nh, inter=Fp, engine="layered")
        if params is not None:
            hs = slice(rank * nh, (rank + 1) * nh)
            layers = [shard_layer_b16(lp, rank, world) for lp in params["layers"]]
            cl = [[(k[hs], v[hs]) for k, v in per_layer] for per_layer in caches]
            self.m = BatchedLlama.from_params(self.lcfg, layers, cl, cache_cap)
        else:
            self.m = BatchedLlama.random(self.lcfg, cache_cap, seed=seed)

    def stage(self, layer: int, stage: int) -> None:
        m = self.m
        _native.check(_native.lib().cfb_llama_b16_layer(
            m.layer_args(m.layers[layer], stage=stage, partial=self.rank > 0), m.stream.cuda_stream))

    def allreduce(self) -> None:
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(self.m.resid, group=self.group)

    def _enqueue(self) -> None:
        for l in range(len(self.m.layers)):
            self.stage(l, 1)
            self.allreduce()
            self.stage(l, 2)
            self.allreduce()
        _native.check(_native.lib().cfb_b16_advance(self.m.pos.data_ptr(), self.m.B, self.m.stream.cuda_stream))

    def step(self) -> None:
        import torch
        self.m._check_room(1)
        with torch.cuda.stream(self.m.stream):
            self._enqueue()
        self.m._advance_host()

    def capture(self) -> None:
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.m.stream):
            self._enqueue()

    def replay(self) -> None:
        import torch
        self.m._check_room(1)
        with torch.cuda.stream(self.m.stream):
            self.graph.replay()
        self.m._advance_host()


# --------------------------------------------------------------------------
# DeepSeek-V2-Lite block, tensor parallel (SURVEY §8(e) caveats): MLA heads
# sharded (W_q / W_up / W_down / W_out per head), the latent cache and W_kv
# replicated (every rank computes the new latent row itself); MoE "TP inside
# experts": every routed and shared expert's intermediate dimension sharded,
# the router replicated (identical inputs -> identical routing on all ranks).
# Exchange steps: one int64 all-reduce of the fixed-point attention head sum
# (exact), one fp32 all-reduce of the block output (rank 0 carries the
# residual + attention, ranks > 0 their MoE partial: CFB_PARTIAL).
# --------------------------------------------------------------------------
def check_tp_deepseek(dims, world: int) -> None:
    if world < 1 or dims.n_heads % world:
        raise DimensionError(f"tensor parallel {world}: n_heads {dims.n_heads} must divide")
    f = dims.inter // world
    if dims.inter % world or f % 8 or (dims.n_shared * f) % 8:
        raise DimensionError(f"tensor parallel {world}: expert width {dims.inter} / {world} must be a multiple of 8")


def deepseek_local_dims(dims, world: int):
    check_tp_deepseek(dims, world)
    return replace(dims, n_heads=dims.n_heads // world, inter=dims.inter // world)


def shard_deepseek(dims, mla_arrays: dict, moe_w: dict, rank: int, world: int):
    """Oracle-format block weights -> this rank's shard: (local dims, MLA
    arrays, MoE weights dict).  Heads [rank*nh/TP, (rank+1)*nh/TP); expert
    intermediate rows [rank*F/TP, (rank+1)*F/TP) of every routed expert and
    the same fraction of the (concatenated) shared expert."""
    ld = deepseek_local_dims(dims, world)
    h0, h1 = rank * ld.n_heads, (rank + 1) * ld.n_heads
    mla = dict(w_q=mla_arrays["w_q"][h0:h1], w_up=mla_arrays["w_up"][h0:h1], w_kv=mla_arrays["w_kv"],
               w_down=mla_arrays["w_down"][h0:h1], w_out=mla_arrays["w_out"][h0:h1],
               kv_cache=mla_arrays["kv_cache"])

    def cut(ex, f):
        lo, hi = rank * f, (rank + 1) * f
        return dict(gate=ex["gate"][lo:hi], up=ex["up"][lo:hi], down=ex["down"][:, lo:hi])

    moe = dict(router=moe_w["router"],
               experts=[cut(moe_w["experts"][e], ld.inter) for e in range(len(moe_w["experts"]))],
               shared=None if moe_w.get("shared") is None else cut(moe_w["shared"], ld.n_shared * ld.inter))
    return ld, mla, moe


class TPDeepSeekBlock:
    """One rank of a tensor-parallel DeepSeek block.  ``reduce_int`` /
    ``reduce_f32`` are the all-reduce(SUM) callables (NCCL in production,
    a device sum in the emulated single-GPU test)."""

    def __init__(self, dims, rank: int, world: int, block, reduce_int=None, reduce_f32=None):
        self.dims, self.rank, self.world, self.block = dims, rank, world, block
        block.partial = rank > 0
        self.reduce_int, self.reduce_f32 = reduce_int, reduce_f32

    @classmethod
    def from_arrays(cls, dims, mla_arrays, moe_w, attn_norm, ffn_norm, rank, world, **kw):
        from .deepseek import DeepSeekBlock
        ld, mla, moe = shard_deepseek(dims, mla_arrays, moe_w, rank, world)
        return cls(dims, rank, world, DeepSeekBlock.from_arrays(ld, mla, moe, attn_norm, ffn_norm), **kw)

    @classmethod
    def random(cls, dims, rank, world, seq_len, seed=0, **kw):
        from .deepseek import DeepSeekBlock
        ld = deepseek_local_dims(dims, world)
        return cls(dims, rank, world, DeepSeekBlock.random(ld, seq_len, seed=seed * 100 + rank), **kw)

    @staticmethod
    def nccl_reducers():
        import torch.distributed as dist
        return (lambda t: dist.all_reduce(t), lambda t: dist.all_reduce(t))

    def launch_attention(self, resid, stream=None) -> None:
        self.block.launch_attention(resid, pdl=True, stream=stream)

    def launch_moe(self, resid, stream=None) -> None:
        b = self.block
        from .moe import moe_launch
        moe_launch(b.moe, b.ws, resid, resid=resid, norm_w=b.ffn_norm, accum_in=b.accum_attn,
                   eps=b.dims.eps, pdl=False, stream=stream, partial=b.partial)

    def launch(self, resid, stream=None) -> None:
        """resid (replicated, [1][D] fp32) <- block(resid) on every rank."""
        self.launch_attention(resid, stream)
        if self.world > 1:
            self.reduce_int(self.block.accum_attn)
        self.launch_moe(resid, stream)
        if self.world > 1:
            self.reduce_f32(resid)
