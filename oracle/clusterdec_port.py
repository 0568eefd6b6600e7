"""numpy restatement of the reference ``clusterdec`` algorithms (TEST ORACLE ONLY).

Everything here is the checker for ``paper_2508_18850_b200``; nothing in the
shipped package imports it.  Each function names the reference file:line it
restates (paths relative to ``/root/reference/pkg/src/clusterdec``).

Storage model (``simcore.py:45-52``, ``simcore.py:94-110``): arithmetic is
float32; with the ``"f16"`` tag every *buffer store* is rounded to the nearest
binary16 value.  The partition-level functions below apply that rounding at
exactly the store points the reference simulator has, so the restated
dataflows reproduce the reference's numbers, and — with ``head_accum="f32"`` —
the GPU kernel's numbers (which accumulate heads in fp32).
"""

from __future__ import annotations

import math

import numpy as np

F32 = "f32"
F16 = "f16"


# --------------------------------------------------------------------------
# storage rounding + seeded inputs
# --------------------------------------------------------------------------

def tag_for_bytes(nbytes: int) -> str:
    """``simcore.py:37-42``: 4 -> f32, 2 -> f16-emulated."""
    return {4: F32, 2: F16}[nbytes]


def rnd(values, tag: str) -> np.ndarray:
    """Store rounding (``simcore.py:45-52``)."""
    a = np.asarray(values, dtype=np.float32)
    return a.astype(np.float16).astype(np.float32) if tag == F16 else a


def _draw(rng: np.random.Generator, shape, scale: float, tag: str) -> np.ndarray:
    """``scenarios.py:108-109``: N(0,1)*scale in float64, cast f32, store-round."""
    return rnd((rng.standard_normal(shape) * scale).astype(np.float32), tag)


def gen_mha(B, D, n_heads, H, S, dtype_bytes=2, seed=0) -> dict:
    """Draw order and scales of ``random_mha_scenario`` (``scenarios.py:112-137``)."""
    rng = np.random.default_rng(seed)
    tag = tag_for_bytes(dtype_bytes)
    out = {}
    out["hidden"] = _draw(rng, (B, D), 1.0, tag)
    out["w_qkv"] = _draw(rng, (n_heads, D, 3 * H), D ** -0.5, tag)
    out["w_out"] = _draw(rng, (n_heads, H, D), H ** -0.5, tag)
    out["k_cache"] = _draw(rng, (n_heads, S, H), 1.0, tag)
    out["v_cache"] = _draw(rng, (n_heads, S, H), 1.0, tag)
    return out


def gen_mla(B, D, n_heads, H, S, rank, dtype_bytes=2, seed=0) -> dict:
    """Draw order and scales of ``random_mla_scenario`` (``scenarios.py:140-165``)."""
    rng = np.random.default_rng(seed)
    tag = tag_for_bytes(dtype_bytes)
    out = {}
    out["hidden"] = _draw(rng, (B, D), 1.0, tag)
    out["w_q"] = _draw(rng, (n_heads, D, H), D ** -0.5, tag)
    out["w_up"] = _draw(rng, (n_heads, H, rank), H ** -0.5, tag)
    out["w_kv"] = _draw(rng, (D, rank), D ** -0.5, tag)
    out["w_down"] = _draw(rng, (n_heads, rank, H), rank ** -0.5, tag)
    out["w_out"] = _draw(rng, (n_heads, H, D), H ** -0.5, tag)
    out["kv_cache"] = _draw(rng, (S, rank), 1.0, tag)
    return out


# --------------------------------------------------------------------------
# dense oracles (oracle.py)
# --------------------------------------------------------------------------

def softmax(s: np.ndarray) -> np.ndarray:
    """``oracle.py:23-27``."""
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def dense_mha(hidden, w_qkv, w_out, k_cache, v_cache) -> np.ndarray:
    """``oracle.py:30-52``: per head softmax(q [K;k_new]^T / sqrt(H)) [V;v_new] W_out."""
    n_heads, _, three_h = w_qkv.shape
    h = three_h // 3
    out = np.zeros((hidden.shape[0], w_out.shape[2]), np.float32)
    for i in range(n_heads):
        q = hidden @ w_qkv[i][:, :h]
        k = np.concatenate([k_cache[i], hidden @ w_qkv[i][:, h:2 * h]], 0)
        v = np.concatenate([v_cache[i], hidden @ w_qkv[i][:, 2 * h:]], 0)
        out += (softmax(q @ k.T / math.sqrt(h)) @ v) @ w_out[i]
    return out.astype(np.float32)


def dense_mha_stats(hidden, w_qkv, k_cache) -> tuple[np.ndarray, np.ndarray]:
    """Global softmax (max, sum) per head and row — the quantities the
    dataflow reports as ``score_max``/``score_sum`` (``dataflows.py:223-224``)."""
    n_heads, _, three_h = w_qkv.shape
    h = three_h // 3
    ms, ls = [], []
    for i in range(n_heads):
        q = hidden @ w_qkv[i][:, :h]
        k = np.concatenate([k_cache[i], hidden @ w_qkv[i][:, h:2 * h]], 0)
        s = q @ k.T / math.sqrt(h)
        m = s.max(axis=1)
        ms.append(m)
        ls.append(np.exp(s - m[:, None]).sum(axis=1))
    return np.array(ms, np.float32), np.array(ls, np.float32)


def dense_mla(hidden, w_q, w_up, w_kv, w_down, w_out, kv_cache, variant="absorbed"):
    """``oracle.py:55-93``; score scale is 1/sqrt(kv_lora_rank) in both forms."""
    rank = w_kv.shape[1]
    scale = 1.0 / math.sqrt(rank)
    lat = np.concatenate([kv_cache, hidden @ w_kv], 0)
    out = np.zeros((hidden.shape[0], w_out.shape[2]), np.float32)
    for i in range(w_q.shape[0]):
        if variant == "absorbed":
            ql = (hidden @ w_q[i]) @ w_up[i]
            head = (softmax(ql @ lat.T * scale) @ lat) @ w_down[i]
        else:
            q = hidden @ w_q[i]
            k = lat @ w_up[i].T
            v = lat @ w_down[i]
            head = softmax(q @ k.T * scale) @ v
        out += head @ w_out[i]
    return out.astype(np.float32)


def silu(x):
    """``oracle.py:100-101``."""
    return x / (1.0 + np.exp(-x))


def ffn(z, w1, w2, w3, activation="silu"):
    """``oracle.py:112-131``: (act(z w1^T) * (z w2^T)) w3^T."""
    if activation == "silu":
        act = silu
    elif activation == "relu":
        act = lambda x: np.maximum(x, 0.0)  # noqa: E731
    elif activation == "identity":
        act = lambda x: x  # noqa: E731
    else:
        from scipy.special import erf
        act = lambda x: 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))  # noqa: E731
    return ((act(z @ w1.T) * (z @ w2.T)) @ w3.T).astype(np.float32)


def naive_dot_rows(a, b):
    """Scalar float64 loops (the independent dual, ``oracle.py:139-151``)."""
    rows, inner = a.shape
    cols = b.shape[1]
    out = np.zeros((rows, cols))
    for r in range(rows):
        for c in range(cols):
            acc = 0.0
            for k in range(inner):
                acc += float(a[r, k]) * float(b[k, c])
            out[r, c] = acc
    return out.astype(np.float32)


# --------------------------------------------------------------------------
# partition-level primitives (dataflows.py / collectives.py)
# --------------------------------------------------------------------------

def segments(S: int, N: int) -> list[tuple[int, int]]:
    """``dataflows.py:109-114``: contiguous ceil(S/N) segments, tail short/empty."""
    if S == 0:
        return [(0, 0)] * N
    step = -(-S // N)
    return [(min(b * step, S), min(b * step + step, S)) for b in range(N)]


def partial_attention(q, k, v):
    """``dataflows.py:71-99``: (A, m, l) over one segment; empty -> (0, -inf, 0)."""
    B = q.shape[0]
    if k.shape[0] == 0:
        return (np.zeros((B, v.shape[1]), np.float32), np.full(B, -np.inf, np.float32),
                np.zeros(B, np.float32))
    s = (q @ k.T) / math.sqrt(k.shape[1])
    m = s.max(axis=1)
    w = np.exp(s - m[:, None])
    return (w @ v).astype(np.float32), m.astype(np.float32), w.sum(axis=1).astype(np.float32)


def merge_stats(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """``collectives.py:31-55``: [maxes|sums] pair merge with the -inf identity."""
    half = a.size // 2
    ma, sa, mb, sb = a[:half], a[half:], b[:half], b[half:]
    m = np.maximum(ma, mb)

    def scaled(mx, s):
        f = np.zeros_like(m, dtype=np.float32)
        ok = ~np.isneginf(mx)
        f[ok] = np.exp(mx[ok] - m[ok])
        return s * f

    return np.concatenate([m, scaled(ma, sa) + scaled(mb, sb)]).astype(np.float32)


OPS = {
    "sum": lambda a, b: a + b,
    "max": np.maximum,
    "softmax_merge": merge_stats,
}


def ring_reduce(bufs: list[np.ndarray], op: str, tag: str) -> list[np.ndarray]:
    """``collectives.py:110-157``: log2(N) lockstep rounds; block b receives from
    (b - stride) mod N, folds ``op(own, received)`` and store-rounds the result."""
    n = len(bufs)
    cur = [rnd(b, tag) for b in bufs]
    stride = 1
    while stride < n:
        snap = [c.copy() for c in cur]
        cur = [rnd(OPS[op](cur[b], rnd(snap[(b - stride) % n], tag)), tag) for b in range(n)]
        stride *= 2
    return cur


def ring_gather(locals_: list[np.ndarray], tag: str) -> list[np.ndarray]:
    """``collectives.py:160-203``: doubling-prefix all-gather; returns each block's
    buffer in the rotated order (segment j of block b = rank (b-j) mod N)."""
    n = len(locals_)
    seg = locals_[0].size
    bufs = []
    for loc in locals_:
        b = np.zeros(n * seg, np.float32)
        b[:seg] = rnd(loc.ravel(), tag)
        bufs.append(b)
    stride = 1
    while stride < n:
        span = seg * stride
        pre = [b[:span].copy() for b in bufs]
        for r in range(n):
            bufs[r][span:2 * span] = pre[(r - stride) % n]
        stride *= 2
    return bufs


def canonicalize(buf: np.ndarray, rank: int, n: int, seg: int) -> np.ndarray:
    """``collectives.py:206-222``: out[r] = in[(rank - r) mod N]."""
    parts = np.asarray(buf).reshape(n, seg)
    return parts[[(rank - r) % n for r in range(n)]].reshape(-1).copy()


def traffic_reduce(size_bytes: int, n: int) -> int:
    """``analysis.py:64-68``: size * log2(N) * N."""
    return size_bytes * (n.bit_length() - 1) * n


def traffic_gather(size_bytes: int, n: int) -> int:
    """``analysis.py:71-80``: size * (N - 1) * N."""
    return size_bytes * (n - 1) * n


def split_token_traffic(B, H, n, dtype_bytes, stats_mode="two_pass") -> dict:
    """Per-cluster stage bytes of split_token (``analysis.py:212-219``)."""
    h = H // n
    t = {"qkv_gather": traffic_gather(B * 3 * h * dtype_bytes, n)}
    if stats_mode == "merged":
        t["stats_merge_reduce"] = traffic_reduce(2 * B * dtype_bytes, n)
    else:
        t["stats_max_reduce"] = traffic_reduce(B * dtype_bytes, n)
        t["stats_sum_reduce"] = traffic_reduce(B * dtype_bytes, n)
    t["attn_out_reduce"] = traffic_reduce(B * H * dtype_bytes, n)
    return t


def fused_mla_traffic(B, H, rank, n, dtype_bytes, stats_mode="two_pass") -> dict:
    """Per-cluster stage bytes of fused_mla (``analysis.py:220-230``)."""
    h, rs = H // n, rank // n
    t = {
        "q_proj_gather": traffic_gather(B * h * dtype_bytes, n),
        "latent_kv_gather": traffic_gather(B * rs * dtype_bytes, n),
        "absorbed_q_gather": traffic_gather(B * rs * dtype_bytes, n),
    }
    if stats_mode == "merged":
        t["stats_merge_reduce"] = traffic_reduce(2 * B * dtype_bytes, n)
    else:
        t["stats_max_reduce"] = traffic_reduce(B * dtype_bytes, n)
        t["stats_sum_reduce"] = traffic_reduce(B * dtype_bytes, n)
    t["attn_out_reduce"] = traffic_reduce(B * rank * dtype_bytes, n)
    t["down_proj_reduce"] = traffic_reduce(B * H * dtype_bytes, n)
    return t


def split_head_traffic(B, D, S, n, dtype_bytes, append=True) -> dict:
    """Per-cluster stage bytes of split_head (``analysis.py:231-236``)."""
    att = S + (B if append else 0)
    return {"score_reduce": traffic_reduce(B * att * dtype_bytes, n),
            "out_proj_reduce": traffic_reduce(B * D * dtype_bytes, n)}


# --------------------------------------------------------------------------
# softmax-stat merge step shared by split_token and fused_mla
# --------------------------------------------------------------------------

def _merge_head_stats(m_loc, l_loc, tag, stats_mode):
    """``dataflows.py:187-227``; returns per-rank (m*, l*) and block-0's pair."""
    n = len(m_loc)
    if stats_mode == "merged":
        red = ring_reduce([np.concatenate([m_loc[b], l_loc[b]]) for b in range(n)],
                          "softmax_merge", tag)
        B = m_loc[0].size
        return red[0][:B].copy(), red[0][B:].copy()
    mx = ring_reduce([m_loc[b] for b in range(n)], "max", tag)
    m_star = mx[0].copy()
    scaled = []
    for b in range(n):
        f = np.where(np.isneginf(m_loc[b]), np.float32(0.0), np.exp(m_loc[b] - m_star))
        scaled.append(l_loc[b] * f)
    sm = ring_reduce(scaled, "sum", tag)
    return m_star, sm[0].copy()


def _rescale(a, m_loc, m_star, l_star, tag):
    """``dataflows.py:230-232``."""
    f = np.where(np.isneginf(m_loc), np.float32(0.0), np.exp(m_loc - m_star)) / l_star
    return rnd(a * f[:, None], tag)


# --------------------------------------------------------------------------
# cluster dataflows
# --------------------------------------------------------------------------

def split_token(arrs: dict, n: int, dtype_bytes: int = 2, stats_mode="two_pass",
                append=True, head_accum="f16_atomic", rope=None):
    """``dataflows.py:235-313`` (split_token, Alg. 3).

    ``head_accum``: ``"f16_atomic"`` reproduces the reference's global-output
    atomics (store-rounded after every per-head add, ``simcore.py:213-229``);
    ``"f32"`` is the GPU kernel's deterministic fp32 head accumulation.
    ``rope``: optional callable(q_full, k_new) -> (q, k) applied after the
    gather (GPU "model mode"; absent from the reference).
    Returns (output, score_max, score_sum).
    """
    tag = tag_for_bytes(dtype_bytes)
    x, W, Wo = arrs["hidden"], arrs["w_qkv"], arrs["w_out"]
    Kc, Vc = arrs["k_cache"], arrs["v_cache"]
    n_heads, D, three_h = W.shape
    H = three_h // 3
    B = x.shape[0]
    h, o = H // n, D // n
    bounds = segments(Kc.shape[1], n)
    out = np.zeros((B, D), np.float32)
    smax = np.zeros((n_heads, B), np.float32)
    ssum = np.zeros((n_heads, B), np.float32)
    for hd in range(n_heads):
        w = W[hd]
        locs = []
        for b in range(n):
            lo, hi = b * h, (b + 1) * h
            locs.append(rnd(np.concatenate(
                [x @ w[:, lo:hi], x @ w[:, H + lo:H + hi], x @ w[:, 2 * H + lo:2 * H + hi]],
                axis=1), tag))
        # every block ends with identical canonical q/k/v (gather is a copy)
        parts = [l.reshape(B, 3 * h) for l in locs]
        q = np.concatenate([p[:, :h] for p in parts], 1)
        kn = np.concatenate([p[:, h:2 * h] for p in parts], 1)
        vn = np.concatenate([p[:, 2 * h:] for p in parts], 1)
        if rope is not None:
            q, kn = rope(q, kn)
        a_loc, m_loc, l_loc = [], [], []
        for b in range(n):
            lo, hi = bounds[b]
            ks, vs = Kc[hd][lo:hi], Vc[hd][lo:hi]
            if append and b == n - 1:
                ks = np.concatenate([ks, kn], 0)
                vs = np.concatenate([vs, vn], 0)
            a, m, l = partial_attention(q, ks, vs)
            a_loc.append(rnd(a, tag))
            m_loc.append(m)
            l_loc.append(l)
        m_star, l_star = _merge_head_stats(m_loc, l_loc, tag, stats_mode)
        smax[hd], ssum[hd] = m_star, l_star
        attn = ring_reduce([_rescale(a_loc[b], m_loc[b], m_star, l_star, tag) for b in range(n)],
                           "sum", tag)
        for b in range(n):
            lo = b * o
            proj = attn[b] @ Wo[hd][:, lo:lo + o]
            if head_accum == "f16_atomic":
                out[:, lo:lo + o] = rnd(out[:, lo:lo + o] + proj, tag)
            else:
                out[:, lo:lo + o] += proj
    return out, smax, ssum


def fused_mla(arrs: dict, n: int, dtype_bytes: int = 2, stats_mode="two_pass",
              append=True, head_accum="f16_atomic"):
    """``dataflows.py:316-429`` (fused MLA, App. B.1).  Returns (out, smax, ssum)."""
    tag = tag_for_bytes(dtype_bytes)
    x = arrs["hidden"]
    Wq, Wup, Wkv, Wdn, Wo, L = (arrs[k] for k in ("w_q", "w_up", "w_kv", "w_down", "w_out",
                                                   "kv_cache"))
    n_heads, D, H = Wq.shape
    R = Wkv.shape[1]
    B = x.shape[0]
    h, rs, o = H // n, R // n, D // n
    bounds = segments(L.shape[0], n)
    out = np.zeros((B, D), np.float32)
    smax = np.zeros((n_heads, B), np.float32)
    ssum = np.zeros((n_heads, B), np.float32)
    for hd in range(n_heads):
        qf = np.concatenate([rnd(x @ Wq[hd][:, b * h:(b + 1) * h], tag) for b in range(n)], 1)
        lat_new = np.concatenate([rnd(x @ Wkv[:, b * rs:(b + 1) * rs], tag) for b in range(n)], 1)
        ql = np.concatenate([rnd(qf @ Wup[hd][:, b * rs:(b + 1) * rs], tag) for b in range(n)], 1)
        a_loc, m_loc, l_loc = [], [], []
        for b in range(n):
            lo, hi = bounds[b]
            seg = L[lo:hi]
            if append and b == n - 1:
                seg = np.concatenate([seg, lat_new], 0)
            a, m, l = partial_attention(ql, seg, seg)
            a_loc.append(rnd(a, tag))
            m_loc.append(m)
            l_loc.append(l)
        m_star, l_star = _merge_head_stats(m_loc, l_loc, tag, stats_mode)
        smax[hd], ssum[hd] = m_star, l_star
        z = ring_reduce([_rescale(a_loc[b], m_loc[b], m_star, l_star, tag) for b in range(n)],
                        "sum", tag)
        down = ring_reduce([rnd(z[b][:, b * rs:(b + 1) * rs] @ Wdn[hd][b * rs:(b + 1) * rs, :], tag)
                            for b in range(n)], "sum", tag)
        for b in range(n):
            lo = b * o
            proj = down[b] @ Wo[hd][:, lo:lo + o]
            if head_accum == "f16_atomic":
                out[:, lo:lo + o] = rnd(out[:, lo:lo + o] + proj, tag)
            else:
                out[:, lo:lo + o] += proj
    return out, smax, ssum


def split_head(arrs: dict, n: int, dtype_bytes: int = 2, append=True,
               head_accum="f16_atomic"):
    """``dataflows.py:432-502`` (split_head, App. B.2).  Returns (out, smax, ssum)."""
    tag = tag_for_bytes(dtype_bytes)
    x, W, Wo = arrs["hidden"], arrs["w_qkv"], arrs["w_out"]
    Kc, Vc = arrs["k_cache"], arrs["v_cache"]
    n_heads, D, three_h = W.shape
    H = three_h // 3
    B = x.shape[0]
    h = H // n
    scale = 1.0 / math.sqrt(H)
    out = np.zeros((B, D), np.float32)
    smax = np.zeros((n_heads, B), np.float32)
    ssum = np.zeros((n_heads, B), np.float32)
    for hd in range(n_heads):
        w = W[hd]
        sl = []
        for b in range(n):
            lo, hi = b * h, (b + 1) * h
            qb, kb, vb = x @ w[:, lo:hi], x @ w[:, H + lo:H + hi], x @ w[:, 2 * H + lo:2 * H + hi]
            ks, vs = Kc[hd][:, lo:hi], Vc[hd][:, lo:hi]
            if append:
                ks = np.concatenate([ks, kb], 0)
                vs = np.concatenate([vs, vb], 0)
            sl.append((qb, ks, vs))
        scores = ring_reduce([rnd((sl[b][0] @ sl[b][1].T) * scale, tag) for b in range(n)],
                             "sum", tag)
        parts = []
        for b in range(n):
            s = scores[b]
            m = s.max(axis=1)
            w_ = np.exp(s - m[:, None])
            l = w_.sum(axis=1)
            att = (w_ / l[:, None]) @ sl[b][2]
            parts.append(rnd(att @ Wo[hd][b * h:(b + 1) * h, :], tag))
            if b == 0:
                smax[hd], ssum[hd] = m, l
        red = ring_reduce(parts, "sum", tag)
        if head_accum == "f16_atomic":
            out = rnd(out + red[0], tag)
        else:
            out += red[0]
    return out, smax, ssum
