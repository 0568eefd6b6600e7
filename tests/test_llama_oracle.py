"""CPU checks of the decode-loop restatements the reference lacks
(oracle/llama_port.py): naive scalar duals and algebraic identities."""

from __future__ import annotations

import math

import numpy as np

from oracle import clusterdec_port as cp
from oracle import llama_port as lp


def test_rmsnorm_against_scalar_loop():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 16)).astype(np.float32)
    g = lp.f16(1 + 0.1 * rng.standard_normal(16))
    got = lp.rmsnorm_f16(x, g, 1e-5)
    for b in range(2):
        ms = sum(float(v) ** 2 for v in x[b]) / 16
        inv = 1.0 / math.sqrt(ms + 1e-5)
        want = [float(np.float16(float(x[b, i]) * inv * float(g[i]))) for i in range(16)]
        np.testing.assert_allclose(got[b], want, rtol=1e-3, atol=1e-3)


def test_rope_is_rotation_and_identity_at_zero():
    cs = lp.rope_table(64, 8)
    x = lp.f16(np.random.default_rng(1).standard_normal((1, 8)))
    np.testing.assert_array_equal(lp.apply_rope(x, 0, cs), x)  # angle 0
    y = lp.apply_rope(x, 17, cs)
    # rotation preserves pair norms (up to f16 storage)
    n0 = x[0, :4] ** 2 + x[0, 4:] ** 2
    n1 = y[0, :4] ** 2 + y[0, 4:] ** 2
    np.testing.assert_allclose(n0, n1, rtol=2e-3)
    # relative-position property of q.k after rotation
    q = lp.f16(np.random.default_rng(2).standard_normal((1, 8)))
    k = lp.f16(np.random.default_rng(3).standard_normal((1, 8)))
    d1 = float((lp.apply_rope(q, 10, cs) @ lp.apply_rope(k, 7, cs).T)[0, 0])
    d2 = float((lp.apply_rope(q, 20, cs) @ lp.apply_rope(k, 17, cs).T)[0, 0])
    assert abs(d1 - d2) < 2e-2


def test_attention_module_reduces_to_dense_oracle():
    """No RoPE: model-mode attention == dense_mha_decode on the same inputs."""
    arr = cp.gen_mha(1, 64, 2, 16, 9, 2, seed=4)
    kc = np.concatenate([arr["k_cache"], np.zeros((2, 1, 16), np.float32)], 1)
    vc = np.concatenate([arr["v_cache"], np.zeros((2, 1, 16), np.float32)], 1)
    out = lp.attention_module(arr["hidden"], arr["w_qkv"], arr["w_out"], kc, vc, 9, 4, None)
    dense = cp.dense_mha(arr["hidden"], arr["w_qkv"], arr["w_out"], arr["k_cache"], arr["v_cache"])
    assert float(np.max(np.abs(out - dense))) <= 2e-2
    # the appended rows are the new token's k/v
    np.testing.assert_allclose(kc[:, 9], lp.f16(arr["hidden"] @ arr["w_qkv"][:, :, 16:32])[:, 0],
                               atol=0)


def test_ffn_block_matches_reference_ffn_without_rounding():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 32)).astype(np.float32)
    g = np.ones(32, np.float32)
    w1 = rng.standard_normal((48, 32)).astype(np.float32) * 0.2
    w2 = rng.standard_normal((48, 32)).astype(np.float32) * 0.2
    w3 = rng.standard_normal((32, 48)).astype(np.float32) * 0.2
    h = lp.rmsnorm_f16(x, g, 1e-5)
    np.testing.assert_allclose(lp.ffn_block(x, g, w1, w2, w3, 1e-5), cp.ffn(h, w1, w2, w3, "silu"),
                               atol=5e-3)
