"""CPU restatement of the DeepSeek-V2-Lite decode block (TEST ORACLE ONLY).

The reference ``clusterdec`` package has the MLA latent attention
(``dataflows.py:316-429`` / ``oracle.py:55-93``, restated in
``clusterdec_port``) but no MoE and no block composition.
The north star (BASELINE.json, config #3) asks for "MLA latent-KV attention +
a fused MoE top-k router plus expert GEMV".  The MoE semantics restated here
are those of DeepSeek-V2(-Lite) as implemented by the ``transformers``
package (``transformers/models/deepseek_v2/modeling_deepseek_v2.py``,
``DeepseekV2Moe.forward`` / ``route_tokens_to_experts`` /
``DeepseekV2Experts.forward`` / ``DeepseekV2MLP``), config values of the
public DeepSeek-V2-Lite checkpoint:

  n_routed_experts 64, num_experts_per_tok 6, n_shared_experts 2,
  moe_intermediate_size 1408, topk_method "greedy", scoring softmax,
  norm_topk_prob False, routed_scaling_factor 1.0, hidden_act silu.

  logits  = h W_r^T                          (fp32; modeling_deepseek_v2.py MoE.forward)
  p       = softmax(logits)                  (fp32)
  idx, w  = top-k of p (greedy)              (ties: lower expert index first)
  y       = sum_k w_k * down_e(f16(silu(gate_e h) * up_e h))       (routed experts)
          + down_s(f16(silu(gate_s h) * up_s h))                    (shared experts:
                                                one MLP of width n_shared * F_e)

``act_store="f16"`` rounds the SwiGLU activation to fp16 — the point where
the GPU kernel stores it (and where an fp16 model stores it);
``act_store="f32"`` is the plain fp32 form, which ``tests/golden/make_moe_golden.py``
pins bit-for-bit-ish (<= 1e-5) against ``transformers``' own module.

Block (restated in the reference's conventions, ``llama_port``):
  h  = f16(rmsnorm(x) * g_attn);  x = x + MLA(h)       (heads summed in fp32)
  h2 = f16(rmsnorm(x) * g_ffn);   x = x + MoE(h2)
"""

from __future__ import annotations

import numpy as np

from . import clusterdec_port as cp
from .llama_port import f16, rmsnorm_f16

# DeepSeek-V2-Lite MoE dims (config.json of the public checkpoint)
LITE = dict(hidden=2048, n_experts=64, top_k=6, inter=1408, n_shared=2)


def gen_moe(D: int, E: int, F: int, n_shared: int, seed: int = 0) -> dict:
    """Seeded fp16-valued MoE weights.  Each expert draws from its own
    generator (seed*1000 + e; shared experts: seed*1000 + E, router: +E+1) so
    a subset can be regenerated without drawing all E experts.  Scales follow
    scenarios.py:129-134 (N(0,1) * fan_in^-1/2)."""
    def draw(s, shape, scale):
        return f16(np.random.default_rng(s).standard_normal(shape, dtype=np.float32) * np.float32(scale))

    w = {"router": draw(seed * 1000 + E + 1, (E, D), D ** -0.5)}
    w["experts"] = LazyExperts(D, F, seed, E)
    if n_shared:
        w["shared"] = gen_expert(D, F * n_shared, seed * 1000 + E)
    else:
        w["shared"] = None
    return w


class LazyExperts:
    """Sequence of the E routed experts, each drawn on first access (the
    oracle at DeepSeek-V2-Lite dims touches only the top-k experts)."""

    def __init__(self, D, F, seed, E):
        self.D, self.F, self.seed, self.E = D, F, seed, E
        self._cache: dict[int, dict] = {}

    def __len__(self):
        return self.E

    def __getitem__(self, e):
        if isinstance(e, slice):
            return [self[i] for i in range(*e.indices(self.E))]
        e = int(e)
        if not 0 <= e < self.E:
            raise IndexError(e)
        if e not in self._cache:
            self._cache[e] = gen_expert(self.D, self.F, self.seed * 1000 + e)
        return self._cache[e]

    def __iter__(self):
        return (self[e] for e in range(self.E))


def gen_expert(D: int, F: int, s: int) -> dict:
    rng = np.random.default_rng(s)
    g = f16(rng.standard_normal((F, D), dtype=np.float32) * np.float32(D ** -0.5))
    u = f16(rng.standard_normal((F, D), dtype=np.float32) * np.float32(D ** -0.5))
    d = f16(rng.standard_normal((D, F), dtype=np.float32) * np.float32(F ** -0.5))
    return {"gate": g, "up": u, "down": d}


def route(h: np.ndarray, w_router: np.ndarray, top_k: int, scale: float = 1.0):
    """Greedy softmax top-k routing (DeepseekV2Moe.route_tokens_to_experts,
    topk_method "greedy").  Returns (idx (B,k) int, weights (B,k) f32, probs
    (B,E) f32, margin (B,) = p_k - p_{k+1}).  Order within a row: descending
    probability, ties toward the lower index."""
    logits = np.asarray(h, np.float32) @ np.asarray(w_router, np.float32).T
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    probs = (e / e.sum(axis=1, keepdims=True)).astype(np.float32)
    B, E = probs.shape
    idx = np.empty((B, top_k), np.int64)
    margin = np.empty(B, np.float32)
    for b in range(B):
        order = np.lexsort((np.arange(E), -probs[b]))
        idx[b] = order[:top_k]
        margin[b] = probs[b, order[top_k - 1]] - (probs[b, order[top_k]] if top_k < E else 0.0)
    wts = (np.take_along_axis(probs, idx, 1) * np.float32(scale)).astype(np.float32)
    return idx, wts, probs, margin


def expert_mlp(h, ex, act_store="f16"):
    """SwiGLU expert (DeepseekV2MLP.forward): down(silu(gate h) * up h)."""
    gate = h @ ex["gate"].T
    up = h @ ex["up"].T
    act = cp.silu(gate) * up
    if act_store == "f16":
        act = f16(act)
    return (act @ ex["down"].T).astype(np.float32)


def moe(h: np.ndarray, w: dict, top_k: int, scale: float = 1.0, act_store="f16"):
    """Routed + shared experts for B token rows (DeepseekV2Moe.forward).
    Returns (y (B,D) f32, idx, weights, margin)."""
    h = np.asarray(h, np.float32)
    idx, wts, _, margin = route(h, w["router"], top_k, scale)
    y = np.zeros_like(h)
    for b in range(h.shape[0]):
        for j in range(top_k):
            y[b] += wts[b, j] * expert_mlp(h[b:b + 1], w["experts"][int(idx[b, j])], act_store)[0]
    if w.get("shared") is not None:
        y += expert_mlp(h, w["shared"], act_store)
    return y.astype(np.float32), idx, wts, margin


def naive_moe(h, w, top_k, scale=1.0):
    """Scalar-loop float64 dual of ``moe(act_store="f32")`` (small dims only)."""
    h = np.asarray(h, np.float64)
    B, D = h.shape
    E = len(w["experts"])
    out = np.zeros((B, D))

    def mlp(x, ex):
        F = ex["gate"].shape[0]
        a = np.zeros(F)
        for f in range(F):
            g = sum(x[d] * float(ex["gate"][f, d]) for d in range(D))
            u = sum(x[d] * float(ex["up"][f, d]) for d in range(D))
            a[f] = g / (1.0 + np.exp(-g)) * u
        return np.array([sum(a[f] * float(ex["down"][o, f]) for f in range(F)) for o in range(D)])

    for b in range(B):
        lg = np.array([sum(h[b, d] * float(w["router"][e, d]) for d in range(D)) for e in range(E)])
        p = np.exp(lg - lg.max())
        p /= p.sum()
        order = sorted(range(E), key=lambda e: (-p[e], e))[:top_k]
        for e in order:
            out[b] += scale * p[e] * mlp(h[b], w["experts"][e])
        if w.get("shared") is not None:
            out[b] += mlp(h[b], w["shared"])
    return out


def block(resid, mla: dict, attn_norm, ffn_norm, moe_w, top_k, n_blocks, eps=1e-6,
          scale=1.0):
    """One DeepSeek-V2-Lite-shaped decode block on B rows of the residual
    stream.  ``mla`` holds the reference MLA weights/cache (``gen_mla`` keys
    minus ``hidden``); the MLA runs with the cluster semantics of
    dataflows.py:316-429 (clusterdec_port.fused_mla) with fp32 head
    accumulation, the kernel's deliberate deviation.  Returns (x_out, info)."""
    x = np.asarray(resid, np.float32)
    h = rmsnorm_f16(x, attn_norm, eps)
    arrs = dict(mla)
    arrs["hidden"] = h
    attn, _, _ = cp.fused_mla(arrs, n_blocks, 2, "two_pass", append=True, head_accum="f32")
    x = (x + attn).astype(np.float32)
    h2 = rmsnorm_f16(x, ffn_norm, eps)
    y, idx, wts, margin = moe(h2, moe_w, top_k, scale)
    return (x + y).astype(np.float32), {"attn": attn, "h2": h2, "idx": idx, "weights": wts,
                                        "margin": margin, "moe": y}
