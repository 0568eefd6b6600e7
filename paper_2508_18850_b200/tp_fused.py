"""Fused tensor-parallel Llama decode: ONE persistent launch per token per
rank, the two all-reduces of every layer and the vocabulary-shard argmax done
inside the step kernel over NVLink peer memory (csrc/decode_step.cu, "tensor
parallel" section, north star (d)).

Rank r holds the Megatron shard of ``tp.shard_params`` (heads, FFN columns,
LM-head rows).  Each block half ends with every CTA red.adding its D/G slice
of the rank's partial sum, as 64-bit fixed point, into every rank's exchange
block (``cfb_tp_xch_bytes``), then all T x G CTAs meet at a cross-rank
counter.  The integer sum is exact and independent of arrival order, so the
result does not depend on which rank finishes first and is bit-identical run
to run - the same property the NCCL int64 all-reduce of ``tp.TPLlamaDecoder``
(the baseline path, kept) has, without its 2L + 1 collective launches.

Peers' exchange blocks are mapped with CUDA IPC (``cfb_ipc_alloc`` /
``cfb_ipc_open``); the 64-byte handles travel over the torch.distributed
group.  ``emulated_ranks`` builds all T ranks inside one process on one GPU
(each on its own stream and a 1/T share of the SMs, peers' blocks addressed
directly): the same kernel code and protocol, used by the single-GPU tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import numpy as np

from . import _native
from .exceptions import DimensionError
from .llama import LlamaConfig, LlamaDecoder
from .tp import check_tp, shard_params

_vp = ctypes.c_void_p


def _bind(L):
    L.cfb_llama_set_tp_fused.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_longlong]
    L.cfb_llama_set_tp_fused.restype = ctypes.c_int
    L.cfb_tp_xch_bytes.argtypes = [ctypes.c_int]
    L.cfb_tp_xch_bytes.restype = ctypes.c_size_t
    L.cfb_ipc_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp), _vp]
    L.cfb_ipc_open.argtypes = [_vp, ctypes.POINTER(_vp)]
    L.cfb_ipc_close.argtypes = [_vp]
    L.cfb_dev_free.argtypes = [_vp]
    return L


def fused_local_config(cfg: LlamaConfig, world: int, cluster: int | None = None) -> LlamaConfig:
    """Per-rank shape of the fused path: the shard of heads / FFN / vocab and
    the persistent engine.  The attention module of a head runs on one
    cluster, so with nh/T heads per rank the cluster grows until the heads
    cover ~64 CTAs (TP2: 16 heads x 4, TP4: 8 x 8, TP8: 4 x 16): the step
    kernel's per-SM stream rate is capped (~50-90 GB/s, tools/ubench/stream_probe),
    so a head on 4 SMs would take as long at TP8 as at TP1 (DESIGN.md section 5,
    profiles/r02/tp_shard_trace.json).  Every choice keeps nh/T <= the
    co-resident clusters of that size (33 / 15 / 7 for N = 4 / 8 / 16).
    `cluster` overrides (the single-GPU emulation shares one GPU between the
    ranks and keeps cfg.cluster)."""
    check_tp(cfg, world)
    eng = cfg.engine if cfg.engine != "layered" else "persistent"
    nh = cfg.n_heads // world
    if cluster is None:
        cluster = cfg.cluster
        while 2 * cluster <= 16 and nh * cluster < 64 and cfg.head_dim % (2 * cluster) == 0:
            cluster *= 2
    return replace(cfg, n_heads=nh, inter=cfg.inter // world, vocab=cfg.vocab // world, engine=eng,
                   cluster=cluster)


class XchBlock:
    """One rank's exchange block (device memory, zeroed) + its IPC handle."""

    def __init__(self, hidden: int):
        L = _bind(_native.lib())
        self.nbytes = int(L.cfb_tp_xch_bytes(hidden))
        self.ptr = _vp()
        self.handle = (ctypes.c_char * 64)()
        _native.check(L.cfb_ipc_alloc(self.nbytes, ctypes.byref(self.ptr), self.handle))
        self._L = L

    def handle_bytes(self) -> bytes:
        return bytes(self.handle)

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            try:
                self._L.cfb_dev_free(self.ptr)
            except Exception:
                pass


class FusedTPLlama:
    """Rank-local decoder of the fused tensor-parallel path.

    Multi-process (one GPU per rank): ``FusedTPLlama(cfg, rank, world, cap,
    group=...)`` exchanges IPC handles over `group` (any torch.distributed
    backend).  Single-process emulation: see ``emulated_ranks``."""

    def __init__(self, cfg: LlamaConfig, rank: int, world: int, cache_cap: int, *, params=None,
                 seed: int = 0, group=None, peers=None, emulated: bool = False, grid: int = 0,
                 timeout_s: float = 10.0):
        if world < 2:
            raise DimensionError("fused tensor parallel needs at least 2 ranks")
        self.cfg, self.rank, self.world = cfg, rank, world
        self.lcfg = fused_local_config(cfg, world, cfg.cluster if emulated else None)
        if params is not None:
            self.eng = LlamaDecoder.from_params(self.lcfg, shard_params(params, rank, world), cache_cap)
        else:
            self.eng = LlamaDecoder.random(self.lcfg, cache_cap, seed=seed, embed_vocab=cfg.vocab)
        L = _bind(_native.lib())
        self._L = L
        self.xch = XchBlock(cfg.hidden)
        self._opened = []
        if peers is None:  # multi-process: gather the IPC handles, open the peers'
            import torch.distributed as dist
            handles = [None] * world
            dist.all_gather_object(handles, self.xch.handle_bytes(), group=group)
            ptrs = []
            for t, h in enumerate(handles):
                if t == rank:
                    ptrs.append(self.xch.ptr.value)
                    continue
                p = _vp()
                hb = (ctypes.c_char * 64).from_buffer_copy(h)
                _native.check(L.cfb_ipc_open(hb, ctypes.byref(p)))
                self._opened.append(p)
                ptrs.append(p.value)
            self._attach(ptrs, emulated=False, grid=grid, timeout_s=timeout_s)
        self._pending = (emulated, grid, timeout_s)

    def _attach(self, ptrs, emulated, grid, timeout_s):
        arr = (_vp * self.world)(*ptrs)
        _native.check(self._L.cfb_llama_set_tp_fused(self.eng._h, self.rank, self.world,
                                                     self.rank * self.lcfg.vocab, arr,
                                                     1 if emulated else 0, grid,
                                                     int(timeout_s * 1e9)))

    # ------------------------------------------------------------ driving
    @property
    def stream(self):
        return self.eng.stream

    @property
    def launches_per_step(self) -> int:
        return self.eng.launches_per_step

    def set_state(self, pos: int, token: int) -> None:
        self.eng.set_state(pos, token)

    def step(self) -> None:
        self.eng.step()

    def capture(self) -> None:
        self.eng.capture()

    def replay(self) -> None:
        self.eng.replay()

    def token(self) -> int:
        return self.eng.token()

    def logits_local(self) -> np.ndarray:
        return self.eng.logits()

    def check(self) -> None:
        self.eng.check()

    def __del__(self):
        for p in getattr(self, "_opened", []):
            try:
                self._L.cfb_ipc_close(p)
            except Exception:
                pass


class EmulatedTP:
    """All `world` ranks of the fused path in one process on one GPU (tests,
    single-GPU evidence): each rank's kernel runs on its own stream on
    `grid` CTAs; peers' exchange blocks are addressed directly."""

    def __init__(self, ranks):
        self.ranks = ranks

    def set_state(self, pos: int, token: int) -> None:
        for r in self.ranks:
            r.set_state(pos, token)

    def step(self) -> None:
        import torch
        for r in self.ranks:  # all ranks' launches in flight together
            r.step()
        for r in self.ranks:
            r.stream.synchronize()
        torch.cuda.synchronize()

    def capture(self) -> None:
        for r in self.ranks:
            r.capture()

    def replay(self) -> None:
        for r in self.ranks:
            r.replay()
        for r in self.ranks:
            r.stream.synchronize()

    def tokens(self) -> list:
        return [r.token() for r in self.ranks]

    def logits(self) -> np.ndarray:
        return np.concatenate([r.logits_local() for r in self.ranks])

    def check(self) -> None:
        for r in self.ranks:
            r.check()


def emulated_grid(cfg: LlamaConfig, world: int) -> int:
    """CTAs per emulated rank so that all ranks are co-resident on one B200:
    a 1/world share of the SMs (cluster engines: of the 33 co-resident
    4-CTA clusters a ~225 KB CTA allows, ncu launch__cluster_max_active)."""
    sms = int(_native.lib().cfb_device_sm_count())
    lcfg = fused_local_config(cfg, world, cfg.cluster)
    if lcfg.engine == "persistent_flat":
        return sms // world
    N = cfg.cluster
    clusters = (sms // N * 7 // 8) // world  # 37 -> 32 slots: margin for GPC fragmentation
    return clusters * N


def emulated_ranks(cfg: LlamaConfig, world: int, cache_cap: int, *, params=None, seed: int = 0,
                   timeout_s: float = 10.0) -> EmulatedTP:
    grid = emulated_grid(cfg, world)
    ranks = [FusedTPLlama(cfg, r, world, cache_cap, params=params, seed=seed, peers=True,
                          emulated=True, grid=grid, timeout_s=timeout_s) for r in range(world)]
    ptrs = [r.xch.ptr.value for r in ranks]
    for r in ranks:
        r._attach(ptrs, emulated=True, grid=grid, timeout_s=timeout_s)
    return EmulatedTP(ranks)
