"""Llama2-family greedy decode on the B200 kernels (north-star config #2).

``LlamaDecoder`` holds the weights and KV cache in HBM in the kernels'
layouts and drives the native engine (``cfb_llama_*`` in ``csrc/llama.cu``):
one step = embed -> n_layers x (split_token attention module with RMSNorm,
RoPE, KV append and residual -> fused SwiGLU FFN with RMSNorm and residual)
-> final RMSNorm + LM head + argmax, captured once into a CUDA graph.

Weights come either from ``random_llama_params`` (numpy, reference draw
conventions of ``scenarios.py:108-137``; used for parity against the CPU
oracle) or are drawn directly on the device in the packed layouts
(``LlamaDecoder.random``; used by the benchmark, where generating 6.7 B
parameters on the host would dominate the run).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .exceptions import DimensionError, SimulationError
from .layouts import gate_up_tiles, qkv_tiles, row_tiles, wo_rows


@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int = 32
    hidden: int = 4096
    n_heads: int = 32
    head_dim: int = 128
    inter: int = 11008
    vocab: int = 32000
    eps: float = 1e-5
    rope_theta: float = 10000.0
    cluster: int = 4
    dtype_bytes: int = 2
    # "persistent": one launch per step on every SM, attention on DSMEM clusters
    # (csrc/decode_step.cu); "persistent_nodsmem": same clusters, gather and
    # exchange through global memory (the paper's without-DSMEM ablation);
    # "persistent_flat": attention split over all SMs, exchange through global
    # memory (A/B); "layered": split_token cluster kernel + fused
    # FFN kernel per layer, PDL-chained (csrc/llama.cu; the tensor-parallel path)
    engine: str = "persistent"

    def weight_bytes(self) -> int:
        """Bytes of every weight a decode step streams (attention + FFN + norms,
        LM head, one embedding row) — SURVEY.md §8(d)."""
        D, F, nb = self.hidden, self.inter, self.dtype_bytes
        per_layer = (D * 3 * self.n_heads * self.head_dim + self.n_heads * self.head_dim * D
                     + 3 * D * F) * nb + 2 * D * nb
        return self.n_layers * per_layer + self.vocab * D * nb + D * nb + D * nb

    def kv_bytes_per_position(self) -> int:
        return self.n_layers * 2 * self.n_heads * self.head_dim * self.dtype_bytes

    def step_bytes(self, ctx: int) -> int:
        """Algorithmic HBM bytes of one decode step at `ctx` cached positions:
        weights + KV read of ctx positions + KV write of the new one."""
        return self.weight_bytes() + self.kv_bytes_per_position() * (ctx + 1)


LLAMA2_7B = LlamaConfig()


class _LlamaConfigC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "n_layers", "hidden", "n_heads", "head_dim",
                                             "inter", "vocab", "cache_cap", "cluster")] + [
        ("eps", ctypes.c_float), ("engine", ctypes.c_int)]


ENGINES = {"layered": 0, "persistent": 1, "persistent_flat": 2, "persistent_nodsmem": 3}


_PP = ctypes.POINTER(ctypes.c_void_p)


class _LlamaWeightsC(ctypes.Structure):
    _fields_ = [("embed", ctypes.c_void_p), ("final_norm", ctypes.c_void_p),
                ("lm_head", ctypes.c_void_p), ("rope_cs", ctypes.c_void_p)] + [
        (n, _PP) for n in ("attn_norm", "w_qkv", "w_out", "ffn_norm", "w_gu", "w_dn",
                           "k_cache", "v_cache")]


def rope_table(max_pos: int, head_dim: int, theta: float) -> np.ndarray:
    """(max_pos, H/2, 2) fp32 (cos, sin) of rotate-half RoPE; angles in fp64."""
    half = head_dim // 2
    inv_freq = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / head_dim)
    ang = np.outer(np.arange(max_pos, dtype=np.float64), inv_freq)
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


def _draw(rng, shape, scale, shift=0.0):
    x = (rng.standard_normal(shape) * scale + shift).astype(np.float32)
    return x.astype(np.float16).astype(np.float32)


def random_llama_layer(cfg: LlamaConfig, seed: int, layer: int, prefill: int = 0) -> dict:
    """Layer `layer` of ``random_llama_params`` on its own (same draws), so a
    32-layer model can be generated, uploaded and checked one layer at a time."""
    D, F, nh, H = cfg.hidden, cfg.inter, cfg.n_heads, cfg.head_dim
    rng = np.random.default_rng(seed * 1000 + layer)
    return dict(
        attn_norm=_draw(rng, (D,), 0.1, 1.0),
        w_qkv=_draw(rng, (nh, D, 3 * H), D ** -0.5),
        w_out=_draw(rng, (nh, H, D), H ** -0.5),
        ffn_norm=_draw(rng, (D,), 0.1, 1.0),
        w1=_draw(rng, (F, D), D ** -0.5),
        w2=_draw(rng, (F, D), D ** -0.5),
        w3=_draw(rng, (D, F), F ** -0.5),
        k_cache=_draw(rng, (nh, prefill, H), 1.0),
        v_cache=_draw(rng, (nh, prefill, H), 1.0))


def random_llama_globals(cfg: LlamaConfig, seed: int) -> dict:
    """Embedding, final norm and LM head of ``random_llama_params``."""
    rng = np.random.default_rng(seed * 1000 + 999)
    D = cfg.hidden
    return dict(embed=_draw(rng, (cfg.vocab, D), 1.0), final_norm=_draw(rng, (D,), 0.1, 1.0),
                lm_head=_draw(rng, (cfg.vocab, D), D ** -0.5))


def random_llama_params(cfg: LlamaConfig, seed: int = 0, prefill: int = 0) -> dict:
    """Seeded numpy parameters in the reference's logical layouts.

    Per layer l: default_rng(seed*1000 + l) draws attn_norm (1 + 0.1 N),
    w_qkv (nh, D, 3H)*D^-1/2, w_out (nh, H, D)*H^-1/2, ffn_norm,
    w1 (F, D)*D^-1/2, w2 (F, D)*D^-1/2, w3 (D, F)*F^-1/2, then the prefilled
    K and V caches (nh, prefill, H) ~ N(0, 1); globals from seed*1000 + 999:
    embed (V, D) ~ N(0, 1), final_norm, lm_head (V, D)*D^-1/2.  All values are
    rounded to fp16."""
    layers = [random_llama_layer(cfg, seed, l, prefill) for l in range(cfg.n_layers)]
    return dict(layers=layers, **random_llama_globals(cfg, seed))


class LlamaDecoder:
    """Device-resident Llama model + KV cache driving the native engine."""

    def __init__(self, cfg: LlamaConfig, cache_cap: int):
        import torch
        if cfg.dtype_bytes != 2:
            raise DimensionError("the decode engine runs fp16 storage only")
        if cfg.head_dim % cfg.cluster or cfg.hidden % cfg.cluster:
            raise DimensionError("head_dim and hidden must be divisible by the cluster size")
        if cfg.engine not in ENGINES:
            raise DimensionError(f"unknown engine {cfg.engine!r} (one of {sorted(ENGINES)})")
        self.cfg = cfg
        self.cache_cap = cache_cap
        self.dev = _native.require_cuda()
        self.torch = torch
        self.layers: list[dict] = []
        self._h = None
        self._keep = []
        self.stream = torch.cuda.Stream(device=self.dev)  # capture needs a non-default stream

    # ------------------------------------------------------------ packing
    def _pack_layer(self, lp: dict) -> dict:
        """Logical numpy layer -> kernel layouts on device (see include/cfb.h)."""
        torch, cfg, dev = self.torch, self.cfg, self.dev
        D, nh, H, F, N = cfg.hidden, cfg.n_heads, cfg.head_dim, cfg.inter, cfg.cluster

        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).half()

        w_qkv = qkv_tiles(t(lp["w_qkv"]), N, H, D)               # row tiles per (head, rank)
        w_out = wo_rows(t(lp["w_out"]).transpose(1, 2).contiguous(), N)  # row tiles per rank
        w_gu = gate_up_tiles(t(lp["w1"]), t(lp["w2"]))            # row tiles (g g u u)
        kc = torch.zeros(nh, self.cache_cap, H, device=dev, dtype=torch.float16)
        vc = torch.zeros_like(kc)
        S0 = lp["k_cache"].shape[1]
        if S0:
            kc[:, :S0] = t(lp["k_cache"])
            vc[:, :S0] = t(lp["v_cache"])
        return dict(attn_norm=t(lp["attn_norm"]), w_qkv=w_qkv, w_out=w_out,
                    ffn_norm=t(lp["ffn_norm"]), w_gu=w_gu, w_dn=self._pack_down(t(lp["w3"])), k_cache=kc,
                    v_cache=vc)

    def _pack_down(self, w3):
        """W_down in the layout of the engine: row tiles (layered FFN kernel) or
        row-block x f-pair blocks (persistent kernel's split-K down projection)."""
        return row_tiles(w3)

    @classmethod
    def from_params(cls, cfg: LlamaConfig, params: dict, cache_cap: int) -> "LlamaDecoder":
        return cls.from_layers(cfg, params["layers"], params, cache_cap)

    @classmethod
    def from_layers(cls, cfg: LlamaConfig, layers, globals_: dict, cache_cap: int) -> "LlamaDecoder":
        """Pack logical layers one at a time (``layers`` may be a generator,
        so host memory holds one fp32 layer at a time) plus the globals
        (embed, final_norm, lm_head)."""
        m = cls(cfg, cache_cap)
        for lp in layers:
            m.layers.append(m._pack_layer(lp))
        m.adopt_globals(globals_)
        return m

    def adopt_globals(self, g: dict) -> None:
        """Upload embed / final_norm / lm_head once every layer is packed, then
        create the native engine."""
        if len(self.layers) != self.cfg.n_layers:
            raise DimensionError(f"got {len(self.layers)} layers, config has {self.cfg.n_layers}")
        torch = self.torch

        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(self.dev).half()

        self.embed, self.final_norm = t(g["embed"]), t(g["final_norm"])
        self.lm_head = row_tiles(t(g["lm_head"]))
        self._finish()

    @classmethod
    def random(cls, cfg: LlamaConfig, cache_cap: int, seed: int = 0,
               embed_vocab: int | None = None) -> "LlamaDecoder":
        """Weights and a full KV cache drawn on the device (torch Philox), packed
        layouts directly.  Scales as random_llama_params.  `embed_vocab`: rows of
        the embedding table when cfg.vocab is a tensor-parallel LM-head shard."""
        m = cls(cfg, cache_cap)
        torch, dev = m.torch, m.dev
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        D, nh, H, F, N = cfg.hidden, cfg.n_heads, cfg.head_dim, cfg.inter, cfg.cluster

        def rnd(shape, scale, shift=0.0):
            x = torch.empty(shape, device=dev, dtype=torch.float16)
            x.normal_(mean=shift, std=scale, generator=g)
            return x

        for _ in range(cfg.n_layers):
            m.layers.append(dict(
                attn_norm=rnd((D,), 0.1, 1.0),
                w_qkv=rnd((nh, N, 3 * H // N // 4, D // 8, 4, 8), D ** -0.5),
                w_out=rnd((nh, N, D // N, H), H ** -0.5), ffn_norm=rnd((D,), 0.1, 1.0),
                w_gu=rnd((F // 2, D // 8, 4, 8), D ** -0.5),
                w_dn=rnd((D // 4, F // 8, 4, 8), F ** -0.5),
                k_cache=rnd((nh, cache_cap, H), 1.0), v_cache=rnd((nh, cache_cap, H), 1.0)))
        m.embed = rnd((embed_vocab or cfg.vocab, D), 1.0)
        m.final_norm = rnd((D,), 0.1, 1.0)
        m.lm_head = rnd((cfg.vocab // 4, D // 8, 4, 8), D ** -0.5)
        m._finish()
        return m

    def _finish(self):
        cfg, torch = self.cfg, self.torch
        self.rope = torch.from_numpy(rope_table(self.cache_cap, cfg.head_dim, cfg.rope_theta)).to(
            self.dev)
        L = cfg.n_layers

        def arr(key):
            a = (ctypes.c_void_p * L)(*[self.layers[i][key].data_ptr() for i in range(L)])
            self._keep.append(a)
            return ctypes.cast(a, _PP)

        c = _LlamaConfigC(dtype=2, n_layers=L, hidden=cfg.hidden, n_heads=cfg.n_heads,
                          head_dim=cfg.head_dim, inter=cfg.inter, vocab=cfg.vocab,
                          cache_cap=self.cache_cap, cluster=cfg.cluster, eps=cfg.eps,
                          engine=ENGINES[cfg.engine])
        w = _LlamaWeightsC(embed=self.embed.data_ptr(), final_norm=self.final_norm.data_ptr(),
                           lm_head=self.lm_head.data_ptr(), rope_cs=self.rope.data_ptr(),
                           attn_norm=arr("attn_norm"), w_qkv=arr("w_qkv"), w_out=arr("w_out"),
                           ffn_norm=arr("ffn_norm"), w_gu=arr("w_gu"), w_dn=arr("w_dn"),
                           k_cache=arr("k_cache"), v_cache=arr("v_cache"))
        L_ = _native.lib()
        L_.cfb_llama_create.argtypes = [ctypes.POINTER(_LlamaConfigC),
                                        ctypes.POINTER(_LlamaWeightsC),
                                        ctypes.POINTER(ctypes.c_void_p)]
        h = ctypes.c_void_p()
        _native.check(L_.cfb_llama_create(c, w, ctypes.byref(h)))
        self._h = h
        for name in ("cfb_llama_step", "cfb_llama_capture", "cfb_llama_replay",
                     "cfb_llama_destroy", "cfb_llama_launches_per_step"):
            getattr(L_, name).argtypes = [ctypes.c_void_p] + ([ctypes.c_void_p]
                                                              if name not in ("cfb_llama_destroy",
                                                                              "cfb_llama_launches_per_step")
                                                              else [])
        L_.cfb_llama_set_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p]
        L_.cfb_llama_read.argtypes = [ctypes.c_void_p] * 4
        L_.cfb_llama_write_token.argtypes = [ctypes.c_void_p] * 3
        self._lib = L_

    # ------------------------------------------------------------ driving
    def _sp(self) -> int:
        return self.stream.cuda_stream

    @property
    def launches_per_step(self) -> int:
        return int(self._lib.cfb_llama_launches_per_step(self._h))

    def set_trace(self, enable: bool = True):
        """Persistent engine: per-CTA globaltimer stamps of every phase boundary
        ([n_layers][grid][8] int64 on device, filled by each step), or None."""
        L_ = self._lib
        L_.cfb_llama_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_int)]
        grid = ctypes.c_int(0)
        if not enable:
            _native.check(L_.cfb_llama_set_trace(self._h, None, ctypes.byref(grid)))
            self.trace = None
            return None
        _native.check(L_.cfb_llama_set_trace(self._h, None, ctypes.byref(grid)))
        self.trace = self.torch.zeros(self.cfg.n_layers, grid.value, 8, dtype=self.torch.int64,
                                      device=self.dev)
        _native.check(L_.cfb_llama_set_trace(self._h, self.trace.data_ptr(), ctypes.byref(grid)))
        return self.trace

    def set_l2_prefetch(self, nbytes: int) -> None:
        """Persistent engines: bytes per CTA of the next phase prefetched into L2
        (past the smem ring) at each grid barrier; capture again afterwards."""
        L_ = self._lib
        L_.cfb_llama_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]
        _native.check(L_.cfb_llama_set_option(self._h, 1, int(nbytes)))

    def set_plain_launch(self, on: bool = True) -> None:
        """Persistent engines: launch without the cooperative attribute (ncu)."""
        L_ = self._lib
        L_.cfb_llama_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]
        _native.check(L_.cfb_llama_set_option(self._h, 2, 1 if on else 0))

    def set_pool_tiles(self, per_cta: int) -> None:
        """Persistent engines: work-stolen gate/up tiles per CTA (0 = 4)."""
        L_ = self._lib
        L_.cfb_llama_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]
        _native.check(L_.cfb_llama_set_option(self._h, 4, int(per_cta)))

    def set_ring_slots(self, spw: int) -> None:
        """Persistent engines: 8 KB ring slots per consumer warp (1..3; 0 =
        the deepest ring that fits); capture again afterwards."""
        L_ = self._lib
        L_.cfb_llama_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]
        _native.check(L_.cfb_llama_set_option(self._h, 3, int(spw)))

    def page_kv(self, reserve: int | None = None, n_pages: int | None = None, shuffle: bool = True,
                seed: int = 0, layout: str = "head_major"):
        """Move the KV caches into a paged pool and re-create the engine on it
        (persistent cluster engines; SURVEY §8(f) rank 4 at batch 1).

        Pages hold 128 positions; a block table [max_pages] (-1 = not
        reserved) maps logical to physical pages.  ``layout``:
        "page_major" is the batched path's ``PagedKVPool`` ([n_pages][n_heads]
        [128][128] per layer, prefill writer ``cfb_b16_kv_write``);
        "head_major" (``HeadMajorKVPool``, [n_heads][n_pages][128][128]) keeps
        each head's pages in one region, so a CTA's rows stay within a few
        GPU memory pages whatever the page order.  Positions 0 .. reserve-1
        (default: the whole cache_cap) get pages, taken in a shuffled order when
        ``shuffle`` so logical and physical pages differ; ``pool.reserve(0, n)``
        adds more between steps.  A step whose new row lands on an unreserved
        page does nothing and ``check()`` raises.  Call before ``capture``."""
        from .batched import PAGE, HeadMajorKVPool, PagedKVPool
        torch, cfg = self.torch, self.cfg
        if cfg.engine not in ("persistent", "persistent_nodsmem"):
            raise DimensionError("paged KV needs a persistent cluster engine")
        if layout not in ("head_major", "page_major"):
            raise DimensionError(f"unknown KV page layout {layout!r}")
        if getattr(self, "kv_pool", None) is not None:
            raise DimensionError("the KV cache is already paged")
        max_pages = -(-self.cache_cap // PAGE)
        cls = HeadMajorKVPool if layout == "head_major" else PagedKVPool
        pool = cls(cfg, n_pages or max_pages, max_pages, self.dev, n_seq=1)
        if shuffle:
            rng = np.random.default_rng(seed)
            pool.free = [int(x) for x in rng.permutation(pool.n_pages)]
        n = self.cache_cap if reserve is None else reserve
        pool.reserve(0, n)
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(self.stream)
        rows = min(n, self.cache_cap)
        for l, lay in enumerate(self.layers):
            pool.write(l, 0, 0, lay["k_cache"][:, :rows], lay["v_cache"][:, :rows], stream=cur)
            lay["k_cache"], lay["v_cache"] = pool.k[l], pool.v[l]
        torch.cuda.synchronize()
        if self._h is not None:
            self._lib.cfb_llama_destroy(self._h)
            self._h = None
        self._finish()
        H = cfg.head_dim
        if layout == "head_major":
            pstride, hstride = PAGE * H, pool.n_pages * PAGE * H
        else:
            pstride, hstride = cfg.n_heads * PAGE * H, PAGE * H
        L_ = self._lib
        L_.cfb_llama_set_kv_pages.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                              ctypes.c_longlong, ctypes.c_longlong]
        _native.check(L_.cfb_llama_set_kv_pages(self._h, pool.table.data_ptr(), max_pages, pstride, hstride))
        self.kv_pool = pool
        return pool

    def kv_rows(self, layer: int, pos: int):
        """(k, v) rows at position ``pos`` of every head, (n_heads, head_dim) fp16
        on the device, whichever layout the cache has."""
        pool = getattr(self, "kv_pool", None)
        if pool is None:
            return self.layers[layer]["k_cache"][:, pos], self.layers[layer]["v_cache"][:, pos]
        from .batched import HeadMajorKVPool
        pg = int(pool.host_table[0, pos // 128])
        if isinstance(pool, HeadMajorKVPool):
            return pool.k[layer][:, pg, pos % 128], pool.v[layer][:, pg, pos % 128]
        return pool.k[layer][pg, :, pos % 128], pool.v[layer][pg, :, pos % 128]

    def check(self) -> None:
        """Raise if a step found the cache full (pos + 1 > cache_cap) and skipped."""
        L_ = self._lib
        L_.cfb_llama_check.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]
        err = ctypes.c_int(0)
        _native.check(L_.cfb_llama_check(self._h, ctypes.byref(err), self._sp()))
        if err.value == 2:
            raise SimulationError("fused tensor-parallel step: peers did not arrive in time")
        if err.value:
            raise DimensionError(f"decode position reached the cache capacity {self.cache_cap} "
                                 "(or, paged, a page that is not reserved)")

    def set_state(self, pos: int, token: int) -> None:
        _native.check(self._lib.cfb_llama_set_state(self._h, pos, token, self._sp()))

    def step(self) -> None:
        """Eager launches of one decode step (no graph)."""
        _native.check(self._lib.cfb_llama_step(self._h, self._sp()))

    def capture(self) -> None:
        """Capture one step into a CUDA graph (call step() once before, so
        kernel attributes are configured outside capture)."""
        _native.check(self._lib.cfb_llama_capture(self._h, self._sp()))

    def replay(self) -> None:
        _native.check(self._lib.cfb_llama_replay(self._h, self._sp()))

    def read_token_async(self, host_int32_ptr: int) -> None:
        """Stream-ordered D2H copy of the current token into host memory."""
        _native.check(self._lib.cfb_llama_read(self._h, ctypes.c_void_p(host_int32_ptr), None,
                                               self._sp()))

    def write_token_async(self, host_int32_ptr: int) -> None:
        """Stream-ordered H2D copy of the next input token from host memory."""
        _native.check(self._lib.cfb_llama_write_token(self._h, ctypes.c_void_p(host_int32_ptr),
                                                      self._sp()))

    def token(self) -> int:
        buf = np.zeros(1, np.int32)
        self.read_token_async(buf.ctypes.data)
        self.stream.synchronize()
        return int(buf[0])

    def logits(self) -> np.ndarray:
        buf = np.zeros(self.cfg.vocab, np.float32)
        _native.check(self._lib.cfb_llama_read(self._h, None, ctypes.c_void_p(buf.ctypes.data),
                                               self._sp()))
        self.stream.synchronize()
        return buf

    def generate(self, first_token: int, pos: int, n_tokens: int, use_graph: bool = True) -> list:
        """Greedy decode n_tokens starting at cache position pos."""
        self.set_state(pos, first_token)
        out = []
        if use_graph:
            self.step()
            self.set_state(pos, first_token)
            self.capture()
        for _ in range(n_tokens):
            self.replay() if use_graph else self.step()
            out.append(self.token())
        return out

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            try:
                self._lib.cfb_llama_destroy(self._h)
            except Exception:
                pass
            self._h = None

