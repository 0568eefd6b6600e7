"""CPU restatement of the full decode step around the fused modules (TEST ORACLE ONLY).

The reference has no RoPE, RMSNorm, residual, FFN block composition, LM head
or multi-layer model.  These restatements define the
numerics the GPU engine must reproduce, with the reference's conventions:
fp32 arithmetic on fp16-valued inputs and an fp16 store wherever the GPU
stores to an fp16 buffer (simcore.py:45-52):

  h      = f16((x * (1/sqrt(mean(x^2) + eps))) * g)          RMSNorm -> GEMV input
  q,k,v  = split_token attention module on h (cluster semantics of
           dataflows.py:235-313, clusterdec_port.split_token) with
           q, k_new rotated (rotate-half RoPE) and f16-stored, k_new/v_new
           appended to the cache at position S, heads summed in fp32
  x      = x + attn
  a      = f16(silu(h2 w1^T) * (h2 w2^T)),  h2 = RMSNorm(x)   (oracle.py:112-131)
  x      = x + a w3^T
  logits = RMSNorm(x, g_final) W_lm^T ; token = argmax (first max index)

Parity is pinned by the naive scalar duals in tests/test_llama_oracle.py and by
reduction to the pinned split_token restatement when RoPE/norm are identity.
"""

from __future__ import annotations

import numpy as np

from . import clusterdec_port as cp


def f16(a) -> np.ndarray:
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def rmsnorm_f16(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    x = np.asarray(x, np.float32)
    ms = (x * x).sum(axis=-1, keepdims=True, dtype=np.float32) / np.float32(x.shape[-1])
    inv = np.float32(1.0) / np.sqrt(ms + np.float32(eps))
    return f16((x * inv) * g)


def rope_table(max_pos: int, head_dim: int, theta: float = 10000.0) -> np.ndarray:
    """(max_pos, H/2, 2) float32 (cos, sin); angles in float64."""
    half = head_dim // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


def apply_rope(x: np.ndarray, pos: int, cs: np.ndarray) -> np.ndarray:
    """rotate-half RoPE on (B, H) rows at positions pos + b, f16-stored."""
    B, H = x.shape
    half = H // 2
    out = np.empty_like(x)
    for b in range(B):
        c, s = cs[pos + b, :, 0], cs[pos + b, :, 1]
        x1, x2 = x[b, :half], x[b, half:]
        out[b, :half] = f16(x1 * c - x2 * s)
        out[b, half:] = f16(x2 * c + x1 * s)
    return out


def attention_module(h, w_qkv, w_out, k_cache, v_cache, S, N, cs=None):
    """Model-mode split_token: attends cache[:S] + the new token, appends the
    new K/V rows at cache[S] (in place), returns the fp32 head sum."""
    arrs = {"hidden": h, "w_qkv": w_qkv, "w_out": w_out,
            "k_cache": k_cache[:, :S], "v_cache": v_cache[:, :S]}

    def rope(q, kn):
        if cs is not None:
            q, kn = apply_rope(q, S, cs), apply_rope(kn, S, cs)
        return q, kn

    out, _, _ = cp.split_token(arrs, N, 2, "two_pass", append=True, head_accum="f32", rope=rope)
    H = w_qkv.shape[2] // 3
    n_heads = w_qkv.shape[0]
    B = h.shape[0]
    hN = H // N
    for hd in range(n_heads):
        w = w_qkv[hd]
        v = np.concatenate([f16(h @ w[:, 2 * H + r * hN:2 * H + (r + 1) * hN]) for r in range(N)], 1)
        k = np.concatenate([f16(h @ w[:, H + r * hN:H + (r + 1) * hN]) for r in range(N)], 1)
        if cs is not None:
            k = apply_rope(k, S, cs)
        k_cache[hd, S:S + B] = k
        v_cache[hd, S:S + B] = v
    return out


def ffn_block(x, g, w1, w2, w3, eps):
    h = rmsnorm_f16(x, g, eps)
    gate = h @ w1.T
    up = h @ w2.T
    act = f16((gate / (np.float32(1.0) + np.exp(-gate))) * up)
    return act @ w3.T


def decode_step(params: dict, caches: list, token: int, pos: int, cfg) -> tuple[np.ndarray, int]:
    """One greedy step; mutates caches (appends at pos).  Returns (logits, token)."""
    cs = params["rope_cs"]
    x = params["embed"][token][None, :].astype(np.float32)
    for l, lp in enumerate(params["layers"]):
        h = rmsnorm_f16(x, lp["attn_norm"], cfg.eps)
        kc, vc = caches[l]
        x = x + attention_module(h, lp["w_qkv"], lp["w_out"], kc, vc, pos, cfg.cluster, cs)
        x = x + ffn_block(x, lp["ffn_norm"], lp["w1"], lp["w2"], lp["w3"], cfg.eps)
    hf = rmsnorm_f16(x, params["final_norm"], cfg.eps)
    logits = (hf @ params["lm_head"].T)[0]
    return logits.astype(np.float32), int(np.argmax(logits))
