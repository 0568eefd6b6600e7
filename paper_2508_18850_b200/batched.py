"""Batched decode of 16 (or 32) independent sequences on tcgen05 (north-star
"tensor cores for the batch>1 projections"; BASELINE config #5 batch 16).
The batch B is the MMA N: 16 or 32 rows per weight block (``batch=``); any
1..B sequences run on it (inactive rows: position -1).

Each sequence has its own KV cache and position.  One layer is
``cfb_llama_b16_layer`` (csrc/tc_gemm.cu + csrc/batch_attn.cu): the QKV, O and
FFN projections run as swap-AB tcgen05 GEMMs (weights = M, the 16 sequences =
N) whose finishing epilogues apply RoPE + cache append, the residual add and
SwiGLU; attention is split-KV flash decoding per (sequence, head).  The
reference's batch semantics (B new tokens of ONE sequence sharing a cache,
oracle.py:45-50) stay with the cluster kernels (`run_fused_mha_decode`); this
module is the serving-style batch of the north star.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .exceptions import DimensionError
from .llama import LlamaConfig, rope_table
from .tc import BATCH, pack_umma

BATCHES = (16, 32)  # MMA N of the batched tcgen05 path


def _check_batch(batch: int) -> int:
    if batch not in BATCHES:
        raise DimensionError(f"the batched tcgen05 path runs batch 16 or 32 (got {batch})")
    return batch


def pack_layer_b16(lp: dict, dev):
    """Logical layer (``random_llama_params`` layout) -> packed tcgen05 weights."""
    import torch

    def t(a):
        if not isinstance(a, torch.Tensor):
            a = torch.from_numpy(np.ascontiguousarray(a, np.float32))
        return a.to(dev).half()

    wqkv = t(lp["w_qkv"])                          # (nh, D, 3H)
    nh, D, H3 = wqkv.shape
    H = H3 // 3
    rows = wqkv.reshape(nh, D, 3, H).permute(2, 0, 3, 1).reshape(3 * nh * H, D)  # [kind][head][i]
    wo = t(lp["w_out"])                            # (nh, H, D)
    w1, w2, w3 = t(lp["w1"]), t(lp["w2"]), t(lp["w3"])
    F = w1.shape[0]
    gu = torch.stack([w1.reshape(-1, 64, D), w2.reshape(-1, 64, D)], 1).reshape(2 * F, D)
    return dict(attn_norm=t(lp["attn_norm"]), ffn_norm=t(lp["ffn_norm"]),
                w_qkv=pack_umma(rows.contiguous()), w_o=pack_umma(wo.reshape(nh * H, D).t().contiguous()),
                w_gu=pack_umma(gu.contiguous()), w_dn=pack_umma(w3))


PAGE = 128  # CFB_KV_PAGE: positions per KV page (= one attention chunk)


# batched projections on CTA pairs sharing each activation block by TMA
# multicast (CFB_TC_PAIR); False = one CTA per run
TC_PAIR = False


class PagedKVPool:
    """Paged KV caches for the n_seq (16 or 32) sequences: per layer a K and a V page pool
    [n_pages][n_heads][128][128] fp16 and one shared block table [n_seq][max_pages]
    (page ids, the same for every layer).  Pages are handed out from a free
    list as sequences grow (``reserve``) and returned by ``release``; the
    device table is refreshed on every change (host-side, between steps)."""

    def __init__(self, cfg: LlamaConfig, n_pages: int, max_pages: int, dev, n_seq: int = BATCH):
        import torch
        self.cfg, self.n_pages, self.max_pages, self.dev = cfg, n_pages, max_pages, dev
        self.n_seq = n_seq
        shape = (n_pages, cfg.n_heads, PAGE, 128)
        self.k = [torch.zeros(shape, device=dev, dtype=torch.float16) for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, device=dev, dtype=torch.float16) for _ in range(cfg.n_layers)]
        self.free = list(range(n_pages))[::-1]
        self.pages = [[] for _ in range(n_seq)]
        # unassigned entries are -1 (never a real page: the kernels drop writes to
        # them instead of aliasing page 0)
        self.host_table = np.full((n_seq, max_pages), -1, np.int32)
        self.table = torch.full((n_seq, max_pages), -1, device=dev, dtype=torch.int32)

    def reserve(self, seq: int, length: int) -> None:
        """Make positions 0 .. length-1 of ``seq`` addressable."""
        need = (length + PAGE - 1) // PAGE
        if need > self.max_pages:
            raise DimensionError(f"sequence {seq}: {length} positions exceed max_pages={self.max_pages}")
        changed = False
        while len(self.pages[seq]) < need:
            if not self.free:
                raise DimensionError("KV page pool exhausted")
            pg = self.free.pop()
            self.host_table[seq, len(self.pages[seq])] = pg
            self.pages[seq].append(pg)
            changed = True
        if changed:
            self._push()

    def _push(self) -> None:
        import torch
        torch.cuda.synchronize()  # no step in flight reads the table
        self.table.copy_(torch_from(self.host_table))
        torch.cuda.synchronize()

    def release(self, seq: int) -> None:
        self.free.extend(reversed(self.pages[seq]))
        self.pages[seq] = []
        self.host_table[seq] = -1
        self._push()

    def capacity(self, seq: int) -> int:
        """Positions of ``seq`` currently addressable (reserved pages x 128)."""
        return len(self.pages[seq]) * PAGE

    def write(self, layer: int, seq: int, start: int, k, v, stream=None) -> None:
        """Prefill writer: rows start .. start+count of ``seq`` from k, v
        (n_heads, count, 128) into the pages (``cfb_b16_kv_write``)."""
        import torch
        k = _half_dev(k, self.dev)
        v = _half_dev(v, self.dev)
        count = k.shape[1]
        self.reserve(seq, start + count)
        if count == 0:
            return
        _native.check(_native.lib().cfb_b16_kv_write(
            self.k[layer].data_ptr(), self.v[layer].data_ptr(), self.table.data_ptr(), self.max_pages, 0,
            self.cfg.n_heads, seq, start, count, k.data_ptr(), v.data_ptr(),
            (stream or torch.cuda.current_stream()).cuda_stream))

    def gather(self, layer: int, seq: int, length: int):
        """Debug view: (k, v) (n_heads, length, 128) of ``seq`` (torch, device)."""
        import torch
        pg = torch.as_tensor(self.pages[seq][:(length + PAGE - 1) // PAGE], device=self.dev, dtype=torch.long)

        def g(pool):
            return pool[pg].permute(1, 0, 2, 3).reshape(self.cfg.n_heads, -1, 128)[:, :length]
        return g(self.k[layer]), g(self.v[layer])


class HeadMajorKVPool(PagedKVPool):
    """Paged KV for the B=1 persistent engine with per-layer pools
    [n_heads][n_pages][128][128] fp16 (head-major: a head's pages share one
    region).  Page bookkeeping (free list, block table, reserve / release) is
    the batched ``PagedKVPool``'s; only the pool layout and the writer differ."""

    def __init__(self, cfg: LlamaConfig, n_pages: int, max_pages: int, dev, n_seq: int = 1):
        import torch
        self.cfg, self.n_pages, self.max_pages, self.dev, self.n_seq = cfg, n_pages, max_pages, dev, n_seq
        shape = (cfg.n_heads, n_pages, PAGE, cfg.head_dim)
        self.k = [torch.zeros(shape, device=dev, dtype=torch.float16) for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, device=dev, dtype=torch.float16) for _ in range(cfg.n_layers)]
        self.free = list(range(n_pages))[::-1]
        self.pages = [[] for _ in range(n_seq)]
        self.host_table = np.full((n_seq, max_pages), -1, np.int32)
        self.table = torch.full((n_seq, max_pages), -1, device=dev, dtype=torch.int32)

    def write(self, layer: int, seq: int, start: int, k, v, stream=None) -> None:
        """Prefill writer: rows start .. start+count of ``seq`` from k, v
        (n_heads, count, 128) device fp16 into their pages (page-sized copies)."""
        k, v = _half_dev(k, self.dev), _half_dev(v, self.dev)
        count = k.shape[1]
        self.reserve(seq, start + count)
        r = 0
        while r < count:
            pos = start + r
            pg, off = int(self.host_table[seq, pos // PAGE]), pos % PAGE
            n = min(PAGE - off, count - r)
            self.k[layer][:, pg, off:off + n] = k[:, r:r + n]
            self.v[layer][:, pg, off:off + n] = v[:, r:r + n]
            r += n

    def gather(self, layer: int, seq: int, length: int):
        import torch
        pg = torch.as_tensor(self.pages[seq][:(length + PAGE - 1) // PAGE], device=self.dev, dtype=torch.long)
        return (self.k[layer][:, pg].reshape(self.cfg.n_heads, -1, self.cfg.head_dim)[:, :length],
                self.v[layer][:, pg].reshape(self.cfg.n_heads, -1, self.cfg.head_dim)[:, :length])

def torch_from(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a))


def _half_dev(a, dev):
    import torch
    if not isinstance(a, torch.Tensor):
        a = torch.from_numpy(np.ascontiguousarray(a, np.float32))
    return a.to(dev).half().contiguous()


class BatchedLlama:
    """Up to 16 independent sequences through a Llama layer stack (tcgen05
    path).  The MMA always runs the 16 rows (N = 16); a sequence whose
    position is -1 is inactive: no RoPE, no KV-cache write, no attention, its
    position does not advance and its output row is undefined - so any batch
    of 1..16 sequences runs on the same kernels (``set_positions`` with fewer
    than 16 entries pads with inactive rows)."""

    def __init__(self, cfg: LlamaConfig, cache_cap: int, layers: list, max_len: int | None = None,
                 pool: PagedKVPool | None = None, batch: int = BATCH):
        import torch
        self.B = B = _check_batch(batch)
        if cfg.head_dim != 128 or cfg.n_heads * 128 > cfg.hidden or cfg.inter % 64:
            raise DimensionError("the batch-16 path needs head_dim 128, n_heads * 128 <= hidden "
                                 "(== unless tensor-parallel) and inter % 64 == 0")
        self.cfg, self.cap = cfg, cache_cap
        self.dev = _native.require_cuda()
        dev = self.dev
        self.layers = layers
        self.max_len = max_len or cache_cap
        D, nh, F = cfg.hidden, cfg.n_heads, cfg.inter
        self.rope = torch.from_numpy(rope_table(cache_cap, 128, cfg.rope_theta)).to(dev)
        self.pos = torch.zeros(B, device=dev, dtype=torch.int32)
        # host mirror of the device positions: every step / replay advances it,
        # and a step is refused before it would write past a sequence's cache
        self.host_pos = np.zeros(B, np.int64)
        self.resid = torch.zeros(B, D, device=dev, dtype=torch.float32)
        nchunks = (self.max_len + 127) // 128
        self.ws = dict(
            xp=torch.zeros(B * max(D, F), device=dev, dtype=torch.float16),
            q16=torch.zeros(B * nh * 128, device=dev, dtype=torch.float16),
            qkv_acc=torch.zeros(B * 3 * nh * 128, device=dev, dtype=torch.int64),
            part=torch.zeros(B * nh * nchunks * 130, device=dev, dtype=torch.float32),
            o_acc=torch.zeros(B * D, device=dev, dtype=torch.int64),
            gu_acc=torch.zeros(B * 2 * F, device=dev, dtype=torch.int64),
            ap=torch.zeros(B * F, device=dev, dtype=torch.float16),
            ticket=torch.zeros((3 * nh * 128 + 2 * D + 2 * F) // 128 + B * nh, device=dev, dtype=torch.int32),
            slots=torch.zeros(int(_native.lib().cfb_b16_slots_floats(D, nh, F, B)), device=dev,
                              dtype=torch.float32))
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = None
        self.pool = pool
        self.tc_pair = TC_PAIR
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- builders
    @classmethod
    def paged(cls, cfg: LlamaConfig, layers_params: list, caches: list, max_len: int,
              n_pages: int | None = None, shuffle_seed: int | None = None, batch: int = BATCH) -> "BatchedLlama":
        """Like ``from_params`` but the KV caches live in a ``PagedKVPool``
        (prefill written through ``cfb_b16_kv_write``); positions up to
        ``max_len`` are addressable.  ``n_pages`` defaults to what 16 sequences
        of ``max_len`` need."""
        dev = _native.require_cuda()
        maxp = (max_len + PAGE - 1) // PAGE
        pool = PagedKVPool(cfg, n_pages or batch * maxp, maxp, dev, n_seq=batch)
        if shuffle_seed is not None:  # non-monotonic page ids (tests)
            pool.free = [int(x) for x in np.random.default_rng(shuffle_seed).permutation(pool.n_pages)]
        layers = [pack_layer_b16(lp_, dev) for lp_ in layers_params]
        for li, (L, cl) in enumerate(zip(layers, caches)):
            L["k_cache"], L["v_cache"] = pool.k[li], pool.v[li]
            for n, (k, v) in enumerate(cl):
                pool.write(li, n, 0, k, v)
        return cls(cfg, max_len, layers, max_len, pool=pool, batch=batch)

    @classmethod
    def random_paged(cls, cfg: LlamaConfig, max_len: int, seed: int = 0, shuffle: bool = True,
                     batch: int = BATCH) -> "BatchedLlama":
        """Device-drawn weights over a paged pool whose pages are fully drawn;
        every sequence gets max_len positions of pages (shuffled page ids)."""
        import torch
        m = cls.random(cfg, cache_cap=1, seed=seed, batch=batch)
        dev = m.dev
        maxp = (max_len + PAGE - 1) // PAGE
        pool = PagedKVPool(cfg, batch * maxp, maxp, dev, n_seq=batch)
        if shuffle:
            rng = np.random.default_rng(seed)
            pool.free = [int(x) for x in rng.permutation(pool.n_pages)]
        g = torch.Generator(device=dev)
        g.manual_seed(seed + 7)
        for li, L in enumerate(m.layers):
            pool.k[li].normal_(generator=g)
            pool.v[li].normal_(generator=g)
            L["k_cache"], L["v_cache"] = pool.k[li], pool.v[li]
        for n in range(batch):
            pool.reserve(n, max_len)
        return cls(cfg, max_len, m.layers, max_len, pool=pool, batch=batch)
    @classmethod
    def from_params(cls, cfg: LlamaConfig, layers_params: list, caches: list, cache_cap: int,
                    max_len: int | None = None, batch: int = BATCH) -> "BatchedLlama":
        """layers_params: logical per-layer weights; caches[l] = list of <= batch
        (k (nh, S_n, H), v) numpy prefixes, one per sequence."""
        import torch
        dev = _native.require_cuda()
        layers = []
        for lp_, cl in zip(layers_params, caches):
            L = pack_layer_b16(lp_, dev)
            kc = torch.zeros(batch, cfg.n_heads, cache_cap, 128, device=dev, dtype=torch.float16)
            vc = torch.zeros_like(kc)
            for n, (k, v) in enumerate(cl):
                S = k.shape[1]
                if S:
                    kc[n, :, :S] = torch.from_numpy(np.ascontiguousarray(k, np.float32)).to(dev).half()
                    vc[n, :, :S] = torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(dev).half()
            L["k_cache"], L["v_cache"] = kc, vc
            layers.append(L)
        return cls(cfg, cache_cap, layers, max_len, batch=batch)

    @classmethod
    def random(cls, cfg: LlamaConfig, cache_cap: int, seed: int = 0, batch: int = BATCH) -> "BatchedLlama":
        """Device-drawn packed weights and full KV caches (benchmarks)."""
        import torch
        dev = _native.require_cuda()
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        D, nh, F = cfg.hidden, cfg.n_heads, cfg.inter

        def rnd(shape, scale, shift=0.0):
            x = torch.empty(shape, device=dev, dtype=torch.float16)
            x.normal_(mean=shift, std=scale, generator=g)
            return x

        layers = []
        for _ in range(cfg.n_layers):
            layers.append(dict(
                attn_norm=rnd((D,), 0.1, 1.0), ffn_norm=rnd((D,), 0.1, 1.0),
                w_qkv=rnd((3 * nh, D // 64, 4, 2, 16, 8, 8), D ** -0.5),
                w_o=rnd((D // 128, 2 * nh, 4, 2, 16, 8, 8), (nh * 128) ** -0.5),
                w_gu=rnd((2 * F // 128, D // 64, 4, 2, 16, 8, 8), D ** -0.5),
                w_dn=rnd((D // 128, F // 64, 4, 2, 16, 8, 8), F ** -0.5),
                k_cache=rnd((batch, nh, cache_cap, 128), 1.0),
                v_cache=rnd((batch, nh, cache_cap, 128), 1.0)))
        return cls(cfg, cache_cap, layers, batch=batch)

    # ---------------------------------------------------------------- running
    def layer_args(self, L: dict, stage: int = 0, partial: bool = False):
        cfg, w = self.cfg, self.ws
        return _native.B16LayerArgs(
            hidden=cfg.hidden, n_heads=cfg.n_heads, inter=cfg.inter, cache_cap=self.cap,
            max_len=self.max_len, flags=_native.PDL | (_native.PARTIAL if partial else 0) | (_native.TC_PAIR if self.tc_pair else 0),
            stage=stage,
            eps=cfg.eps, resid=self.resid.data_ptr(),
            attn_norm=L["attn_norm"].data_ptr(), ffn_norm=L["ffn_norm"].data_ptr(),
            w_qkv=L["w_qkv"].data_ptr(), w_o=L["w_o"].data_ptr(), w_gu=L["w_gu"].data_ptr(),
            w_dn=L["w_dn"].data_ptr(), k_cache=L["k_cache"].data_ptr(),
            v_cache=L["v_cache"].data_ptr(), rope_cs=self.rope.data_ptr(), pos=self.pos.data_ptr(),
            xp=w["xp"].data_ptr(), q16=w["q16"].data_ptr(), qkv_acc=w["qkv_acc"].data_ptr(),
            part=w["part"].data_ptr(), o_acc=w["o_acc"].data_ptr(), gu_acc=w["gu_acc"].data_ptr(),
            ap=w["ap"].data_ptr(), ticket=w["ticket"].data_ptr(),
            block_table=self.pool.table.data_ptr() if self.pool else None,
            max_pages=self.pool.max_pages if self.pool else 0, batch=self.B, slots=w["slots"].data_ptr())

    def _enqueue(self, advance: bool = True) -> None:
        L_ = _native.lib()
        sp = self.stream.cuda_stream
        for L in self.layers:
            _native.check(L_.cfb_llama_b16_layer(self.layer_args(L), sp))
        if advance:
            _native.check(L_.cfb_b16_advance(self.pos.data_ptr(), self.B, sp))

    @property
    def active(self) -> np.ndarray:
        """Indices of the active sequences (position >= 0)."""
        return np.nonzero(self.host_pos >= 0)[0]

    def _advance_host(self) -> None:
        self.host_pos[self.host_pos >= 0] += 1

    def _limit(self, n: int) -> int:
        """Positions sequence n can hold now: the contiguous cache / max_len, or
        its reserved pages."""
        lim = min(self.cap, self.max_len) if self.pool is None else min(self.max_len, self.pool.capacity(n))
        return lim

    def _check_room(self, steps: int = 1) -> None:
        """Raise before a step would append past a sequence's cache."""
        for n in self.active:
            if int(self.host_pos[n]) + steps > self._limit(n):
                raise DimensionError(
                    f"sequence {n}: position {int(self.host_pos[n])} + {steps} step(s) exceeds its "
                    f"cache ({self._limit(n)} positions{'; reserve() more pages' if self.pool else ''})")

    def set_positions(self, pos) -> None:
        import torch
        pos = np.asarray(pos, np.int64).reshape(-1)
        if not 1 <= pos.shape[0] <= self.B or (pos < -1).any() or not (pos >= 0).any():
            raise DimensionError(f"set_positions needs 1..{self.B} positions (>= 0, or -1 = inactive), "
                                 "at least one active")
        pos = np.concatenate([pos, np.full(self.B - pos.shape[0], -1, np.int64)])
        if self.pool:  # the new token's page must exist
            for n, p in enumerate(pos):
                if p >= 0:
                    self.pool.reserve(n, int(p) + 1)
        self.host_pos = pos.copy()
        self._check_room(1)
        self.pos.copy_(torch.as_tensor(pos.astype(np.int32)))
        torch.cuda.synchronize()

    def reserve(self, steps: int) -> None:
        """Paged mode: make the next ``steps`` positions of every sequence
        addressable (call before replaying a captured graph that far)."""
        if self.pool:
            for n in self.active:
                self.pool.reserve(n, int(self.host_pos[n]) + steps)

    def step(self, advance: bool = True) -> None:
        """resid <- the layer stack applied to resid for all active sequences."""
        self._check_room(1)
        self._enqueue(advance)
        if advance:
            self._advance_host()

    def capture(self) -> None:
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._enqueue(True)

    def replay(self) -> None:
        import torch
        self._check_room(1)
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        self._advance_host()  # every captured step advances the active positions

    # ---------------------------------------------------------------- greedy decode
    def set_head(self, embed, final_norm, lm_head) -> None:
        """Embedding table (V, D), final norm (D,), LM head (V, D): logical
        numpy / torch arrays; the LM head is packed for tcgen05."""
        import torch
        dev = self.dev

        def t(a):
            if not isinstance(a, torch.Tensor):
                a = torch.from_numpy(np.ascontiguousarray(a, np.float32))
            return a.to(dev).half()

        self.embed, self.final_norm = t(embed), t(final_norm)
        lm = t(lm_head)
        self.V = lm.shape[0]
        self.lm = pack_umma(lm)
        self.tokens = torch.zeros(self.B, device=dev, dtype=torch.int32)
        self.logits = torch.zeros(self.B, self.V, device=dev, dtype=torch.float32)
        self.lm_acc = torch.zeros(self.B * self.V, device=dev, dtype=torch.int64)
        self.arg_scratch = torch.zeros(65 * 32, device=dev, dtype=torch.int64)
        torch.cuda.synchronize()

    def random_head(self, vocab: int, seed: int = 1) -> None:
        """Device-drawn embedding / final norm / packed LM head (benchmarks)."""
        import torch
        dev, D = self.dev, self.cfg.hidden
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def rnd(shape, scale, shift=0.0):
            x = torch.empty(shape, device=dev, dtype=torch.float16)
            x.normal_(mean=shift, std=scale, generator=g)
            return x

        self.embed, self.final_norm = rnd((vocab, D), 1.0), rnd((D,), 0.1, 1.0)
        self.V = vocab
        self.lm = rnd((vocab // 128, D // 64, 4, 2, 16, 8, 8), D ** -0.5)
        self.tokens = torch.zeros(self.B, device=dev, dtype=torch.int32)
        self.logits = torch.zeros(self.B, vocab, device=dev, dtype=torch.float32)
        self.lm_acc = torch.zeros(self.B * vocab, device=dev, dtype=torch.int64)
        self.arg_scratch = torch.zeros(65 * 32, device=dev, dtype=torch.int64)
        torch.cuda.synchronize()

    def _enqueue_decode(self, logits: bool) -> None:
        L_ = _native.lib()
        sp = self.stream.cuda_stream
        cfg = self.cfg
        _native.check(L_.cfb_embed(2, self.embed.data_ptr(), self.tokens.data_ptr(), self.resid.data_ptr(),
                                   self.B, cfg.hidden, sp))
        for L in self.layers:
            _native.check(L_.cfb_llama_b16_layer(self.layer_args(L), sp))
        _native.check(L_.cfb_b16_lm_head(
            self.resid.data_ptr(), self.final_norm.data_ptr(), self.lm.data_ptr(), self.V, cfg.hidden,
            cfg.eps, self.ws["xp"].data_ptr(), self.lm_acc.data_ptr(), self.tokens.data_ptr(),
            self.logits.data_ptr() if logits else None, self.arg_scratch.data_ptr(), self.B, sp))
        _native.check(L_.cfb_b16_advance(self.pos.data_ptr(), self.B, sp))

    def decode_step(self, logits: bool = False) -> None:
        """One greedy step for all 16 sequences: tokens -> embed -> layers ->
        LM head -> argmax -> tokens; positions advance."""
        import torch
        self._check_room(1)
        with torch.cuda.stream(self.stream):
            self._enqueue_decode(logits)
        self._advance_host()

    def capture_decode(self) -> None:
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._enqueue_decode(False)

    def step_bytes(self, ctx: int, head: bool = False) -> int:
        """Algorithmic HBM bytes per step: layer weights once + each sequence's
        KV rows 0..ctx (read) and the new row (written); with ``head`` also the
        LM head, final norm and the 16 embedding rows."""
        cfg = self.cfg
        D, F = cfg.hidden, cfg.inter
        w = cfg.n_layers * (2 * (4 * D * D + 3 * D * F) + 4 * D)
        nb = len(self.active) or self.B
        kv = cfg.n_layers * nb * 2 * D * 2 * (ctx + 2)
        h = 2 * self.V * D + 2 * D + nb * 2 * D if head else 0
        return w + kv + h
