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

``nvls=True`` moves the two sums onto an NVLink SHARP multicast buffer
(``NvlsSums``, csrc/nvls.cu): each slice element is added ONCE with
``multimem.red.add.u64`` on the multicast address - the switch updates every
rank's copy - instead of once per peer; barriers and the argmax stay on the
exchange blocks.  Emulated on one GPU the ranks share one copy (a multicast
object with one member), which is the same sum.
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
    L.cfb_llama_set_tp_nvls.argtypes = [_vp, _vp, _vp]
    L.cfb_tp_nvls_bytes.argtypes = [ctypes.c_int]
    L.cfb_tp_nvls_bytes.restype = ctypes.c_size_t
    L.cfb_nvls_supported.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.cfb_nvls_create.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_vp)]
    L.cfb_nvls_export_fd.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
    L.cfb_nvls_import_fd.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_int,
                                     ctypes.POINTER(_vp)]
    L.cfb_nvls_add_device.argtypes = [_vp, ctypes.c_int]
    L.cfb_nvls_bind.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
    L.cfb_nvls_size.argtypes = [_vp]
    L.cfb_nvls_size.restype = ctypes.c_size_t
    L.cfb_nvls_destroy.argtypes = [_vp]
    return L


def nvls_supported(device: int = 0) -> bool:
    """Whether the GPU can take part in NVLS multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)."""
    L = _bind(_native.lib())
    v = ctypes.c_int(0)
    _native.check(L.cfb_nvls_supported(device, ctypes.byref(v)))
    return bool(v.value)


def nvls_usable(device: int = 0) -> bool:
    """Whether a multicast object can actually be created here (the attribute
    can be set on a GPU whose fabric slice still refuses cuMulticastCreate,
    e.g. a single GPU handed to a container)."""
    if not nvls_supported(device):
        return False
    L = _bind(_native.lib())
    h = _vp()
    if L.cfb_nvls_create(int(L.cfb_tp_nvls_bytes(4096)), 1, ctypes.byref(h)) != 0:
        return False
    L.cfb_nvls_destroy(h)
    return True


class NvlsSums:
    """This rank's copy of a multicast buffer for the fused all-reduce sums:
    ``uc`` (unicast: reads, re-zeroing) and ``mc`` (multicast: multimem.red).

    Single process (``group=None``): a multicast object with one member - the
    emulated ranks share it.  Multi-process: rank 0 creates the object and
    exports a file descriptor, the others import it from rank 0's process
    (pidfd_getfd), every rank adds its device, and after a group barrier binds
    its own zeroed copy."""

    def __init__(self, hidden: int, device: int, *, world: int = 1, rank: int = 0, group=None):
        L = _bind(_native.lib())
        self._L = L
        self.h = _vp()
        self.uc, self.mc = _vp(), _vp()
        nbytes = int(L.cfb_tp_nvls_bytes(hidden))
        if group is None:
            _native.check(L.cfb_nvls_create(nbytes, 1, ctypes.byref(self.h)))
            _native.check(L.cfb_nvls_add_device(self.h, device))
            _native.check(L.cfb_nvls_bind(self.h, device, ctypes.byref(self.uc), ctypes.byref(self.mc)))
            return
        import os
        import torch.distributed as dist

        def agree(status, what, payload=None):
            # every rank learns every rank's status before anyone goes on, so a
            # failure anywhere raises everywhere instead of leaving peers in a barrier
            got = [None] * world
            dist.all_gather_object(got, (status, payload), group=group)
            bad = [r for r, (st, _) in enumerate(got) if st != 0]
            if bad:
                raise RuntimeError(f"NVLS {what} failed on ranks {bad}: {_native.lib().cfb_last_error()!r}")
            return got

        st, mine = 0, None
        if rank == 0:
            st = L.cfb_nvls_create(nbytes, world, ctypes.byref(self.h))
            fd = ctypes.c_int(-1)
            if st == 0:
                st = L.cfb_nvls_export_fd(self.h, ctypes.byref(fd))
            mine = (os.getpid(), fd.value)
        got = agree(st, "create/export", mine)
        st = 0
        if rank != 0:
            pid, fd = got[0][1]
            st = L.cfb_nvls_import_fd(pid, fd, nbytes, world, ctypes.byref(self.h))
        agree(st, "import")
        if rank == 0 and mine[1] >= 0:
            os.close(mine[1])  # every member holds its own reference now
        agree(L.cfb_nvls_add_device(self.h, device), "add_device")  # all adds before any bind
        agree(L.cfb_nvls_bind(self.h, device, ctypes.byref(self.uc), ctypes.byref(self.mc)), "bind")

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            try:
                self._L.cfb_nvls_destroy(self.h)
            except Exception:
                pass


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
                 timeout_s: float = 10.0, nvls: bool = False):
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
            if nvls:
                import torch
                self.nvls = NvlsSums(cfg.hidden, torch.cuda.current_device(), world=world, rank=rank,
                                     group=group)
                self.use_nvls(self.nvls)
        self._pending = (emulated, grid, timeout_s)

    def use_nvls(self, sums) -> None:
        """Route the sums through `sums` (an ``NvlsSums``) or back to the
        peer-memory pushes (None)."""
        _native.check(self._L.cfb_llama_set_tp_nvls(self.eng._h, sums.uc if sums else None,
                                                    sums.mc if sums else None))

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
                   timeout_s: float = 10.0, nvls: bool = False) -> EmulatedTP:
    grid = emulated_grid(cfg, world)
    ranks = [FusedTPLlama(cfg, r, world, cache_cap, params=params, seed=seed, peers=True,
                          emulated=True, grid=grid, timeout_s=timeout_s) for r in range(world)]
    ptrs = [r.xch.ptr.value for r in ranks]
    for r in ranks:
        r._attach(ptrs, emulated=True, grid=grid, timeout_s=timeout_s)
    tp = EmulatedTP(ranks)
    if nvls:  # one multicast copy on this GPU, shared by every emulated rank
        import torch
        tp.nvls = NvlsSums(cfg.hidden, torch.cuda.current_device())
        for r in ranks:
            r.use_nvls(tp.nvls)
    return tp
