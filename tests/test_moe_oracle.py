"""The MoE oracle (oracle/deepseek_port.py) pinned against golden vectors that
``tests/golden/make_moe_golden.py`` produced with ``transformers``' own
``DeepseekV2Moe`` (greedy softmax top-k, shared experts), plus its scalar
float64 dual and the DeepSeek block composition.  CPU only."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import clusterdec_port as cp
from oracle import deepseek_port as dp
from oracle.llama_port import f16

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def moe_golden():
    meta = json.loads((GOLD / "moe_golden.json").read_text())
    return meta, np.load(GOLD / "moe_golden.npz")


def _hidden(case):
    return f16(np.random.default_rng(case["seed"] + 12345).standard_normal(
        (case["B"], case["D"]), dtype=np.float32))


def _wsha(w):
    import hashlib
    h = hashlib.sha256()
    arrs = [w["router"]] + [x for e in w["experts"] for x in (e["gate"], e["up"], e["down"])]
    if w["shared"]:
        arrs += [w["shared"][k] for k in ("gate", "up", "down")]
    for a in arrs:
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


def test_moe_oracle_matches_transformers_golden(moe_golden):
    meta, g = moe_golden
    for c in meta["cases"]:
        w = dp.gen_moe(c["D"], c["E"], c["F"], c["n_shared"], c["seed"])
        h = _hidden(c)
        if c["D"] <= 256:
            np.testing.assert_array_equal(h, g[c["name"] + "/h"])
            assert _wsha(w) == c["w_sha"], c["name"]
        y, idx, _, margin = dp.moe(h, w, c["K"], c["scale"], act_store="f32")
        np.testing.assert_array_equal(np.sort(idx, 1), g[c["name"] + "/idx"])
        ref = g[c["name"] + "/out"]
        err = float(np.max(np.abs(y - ref)))
        assert err <= 2e-5 * max(1.0, float(np.max(np.abs(ref)))), (c["name"], err)
        assert np.all(margin > 0)


def test_moe_oracle_f16_activation_store_is_within_tolerance(moe_golden):
    meta, g = moe_golden
    for c in meta["cases"]:
        if c["D"] > 512:
            continue
        w = dp.gen_moe(c["D"], c["E"], c["F"], c["n_shared"], c["seed"])
        y16, *_ = dp.moe(_hidden(c), w, c["K"], c["scale"], act_store="f16")
        assert float(np.max(np.abs(y16 - g[c["name"] + "/out"]))) <= 2e-2


def test_moe_oracle_matches_scalar_dual():
    w = dp.gen_moe(16, 6, 8, 1, seed=11)
    h = f16(np.random.default_rng(3).standard_normal((2, 16), dtype=np.float32))
    y, *_ = dp.moe(h, w, 3, 1.5, act_store="f32")
    np.testing.assert_allclose(y, dp.naive_moe(h, w, 3, 1.5), atol=1e-5, rtol=0)


def test_route_ties_break_to_lower_index_and_weights_are_probs():
    h = np.ones((1, 4), np.float32)
    wr = np.array([[1, 0, 0, 0], [0, 0, 0, 2], [0, 1, 0, 0], [0, 0, 0, 0]], np.float32)
    idx, wts, probs, margin = dp.route(h, wr, 2)
    assert idx.tolist() == [[1, 0]]      # logit 2, then the 1-1-tie between experts 0 and 2
    np.testing.assert_allclose(wts[0], probs[0, [1, 0]])
    assert margin[0] == 0.0              # the tie is visible to callers


def test_lazy_experts_equal_eager_draws():
    w = dp.gen_moe(32, 5, 8, 2, seed=4)
    e3 = dp.gen_expert(32, 8, 4 * 1000 + 3)
    for k in ("gate", "up", "down"):
        np.testing.assert_array_equal(w["experts"][3][k], e3[k])
    assert len(list(w["experts"])) == 5


def test_block_composition_reduces_to_parts():
    """block() = residual + MLA(rmsnorm) then residual + MoE(rmsnorm), with the
    MLA restated by the pinned fused_mla restatement."""
    rng = np.random.default_rng(0)
    D, nh, H, R, S = 64, 2, 16, 32, 9
    mla = cp.gen_mla(1, D, nh, H, S, R, 2, seed=5)
    mla.pop("hidden")
    x = rng.standard_normal((1, D)).astype(np.float32)
    ga = f16(1 + 0.1 * rng.standard_normal(D))
    gf = f16(1 + 0.1 * rng.standard_normal(D))
    w = dp.gen_moe(D, 8, 16, 2, seed=1)
    out, info = dp.block(x, mla, ga, gf, w, 2, n_blocks=2)
    from oracle.llama_port import rmsnorm_f16
    attn = cp.dense_mla(rmsnorm_f16(x, ga, 1e-6), *(mla[k] for k in
                        ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")))
    assert float(np.max(np.abs(info["attn"] - attn))) <= 2e-2
    x1 = x + info["attn"]
    y, *_ = dp.moe(rmsnorm_f16(x1, gf, 1e-6), w, 2)
    np.testing.assert_allclose(out, x1 + y, atol=1e-6, rtol=0)
