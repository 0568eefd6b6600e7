"""Pin the CPU oracle (``oracle/clusterdec_port.py``) to the reference's golden vectors.

The fixtures were produced by running the real reference (``make_golden.py``);
these tests run on CPU with no reference present.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import clusterdec_port as cp


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def _inputs(case):
    d = case["dims"]
    if case["kind"] == "fused_mla":
        return cp.gen_mla(d["B"], d["D"], d["n_heads"], d["H"], d["S"], d["rank"],
                          d["dtype_bytes"], case["seed"])
    if case["kind"] == "split_token_preappended":
        base = cp.gen_mha(d["B"], d["D"], d["n_heads"], d["H"], d["S"] - d["B"],
                          d["dtype_bytes"], case["seed"])
        return preappend(base, d["dtype_bytes"])
    return cp.gen_mha(d["B"], d["D"], d["n_heads"], d["H"], d["S"], d["dtype_bytes"],
                      case["seed"])


def preappend(arrs, dtype_bytes):
    """``scenarios.py:168-207``: cache with the new token's K/V pre-appended."""
    tag = cp.tag_for_bytes(dtype_bytes)
    x, W = arrs["hidden"], arrs["w_qkv"]
    H = W.shape[2] // 3
    new = cp.rnd(np.stack([x @ W[i][:, H:] for i in range(W.shape[0])]), tag)
    out = dict(arrs)
    out["k_cache"] = np.concatenate([arrs["k_cache"], new[:, :, :H]], 1)
    out["v_cache"] = np.concatenate([arrs["v_cache"], new[:, :, H:]], 1)
    return out


def _small_cases(meta):
    return [c for c in meta["cases"] if not c["name"].startswith(("llama", "dsv2"))]


def test_generators_bit_exact(golden):
    meta, _ = golden
    for case in _small_cases(meta):
        arrs = _inputs(case)
        for k, h in case["input_sha"].items():
            assert _sha(arrs[k]) == h, (case["name"], k)


@pytest.mark.parametrize("prefix", ["llama2h_n4", "llama_full_s1k_n4", "dsv2_full_s1k_n4"])
def test_generators_bit_exact_production_dims(golden, prefix):
    meta, _ = golden
    case = next(c for c in meta["cases"] if c["name"] == prefix)
    arrs = _inputs(case)
    for k, h in case["input_sha"].items():
        assert _sha(arrs[k]) == h, k


def _run_port(case, arrs, head_accum="f16_atomic"):
    d, n = case["dims"], case["n_blocks"]
    mode = case.get("stats_mode", "two_pass")
    if case["kind"] in ("split_token", "split_token_preappended"):
        return cp.split_token(arrs, n, d["dtype_bytes"], mode,
                              append=case.get("append_new_token", True), head_accum=head_accum)
    if case["kind"] == "fused_mla":
        return cp.fused_mla(arrs, n, d["dtype_bytes"], mode, head_accum=head_accum)
    return cp.split_head(arrs, n, d["dtype_bytes"], head_accum=head_accum)


def test_dataflow_restatement_matches_reference(golden):
    meta, g = golden
    worst = {}
    for case in _small_cases(meta):
        if "stage_traffic" not in case:
            continue
        arrs = _inputs(case)
        out, smax, ssum = _run_port(case, arrs)
        name = case["name"]
        tol = 1e-6 if case["dims"]["dtype_bytes"] == 4 else 2e-3
        err = float(np.max(np.abs(out - g[f"{name}/output"]))) if out.size else 0.0
        worst[case["kind"]] = max(worst.get(case["kind"], 0.0), err)
        assert err <= tol, (name, err)
        np.testing.assert_allclose(smax, g[f"{name}/score_max"], rtol=0, atol=tol)
        np.testing.assert_allclose(ssum, g[f"{name}/score_sum"], rtol=tol, atol=tol)
    assert set(worst) >= {"split_token", "split_head", "fused_mla", "split_token_preappended"}


def test_stage_traffic_formulas_match_reference_ledger(golden):
    meta, _ = golden
    for case in meta["cases"]:
        if "stage_traffic" not in case:
            continue
        d, n = case["dims"], case["n_blocks"]
        mode = case.get("stats_mode", "two_pass")
        if case["kind"].startswith("split_token"):
            per = cp.split_token_traffic(d["B"], d["H"], n, d["dtype_bytes"], mode)
        elif case["kind"] == "fused_mla":
            per = cp.fused_mla_traffic(d["B"], d["H"], d["rank"], n, d["dtype_bytes"], mode)
        else:
            per = cp.split_head_traffic(d["B"], d["D"], d["S"], n, d["dtype_bytes"])
        if n == 1:
            assert case["dsmem_bytes"] == 0
            continue
        want = {k: v * d["n_heads"] for k, v in per.items()}
        assert case["stage_traffic"] == want, case["name"]


def test_dense_oracles_match_reference(golden):
    meta, g = golden
    for case in _small_cases(meta):
        name = case["name"]
        if f"{name}/dense" in g.files:
            a = _inputs(case)
            got = cp.dense_mha(a["hidden"], a["w_qkv"], a["w_out"], a["k_cache"], a["v_cache"])
            np.testing.assert_allclose(got, g[f"{name}/dense"], atol=1e-6, rtol=0)
        if f"{name}/dense_absorbed" in g.files:
            a = _inputs(case)
            args = [a[k] for k in ("hidden", "w_q", "w_up", "w_kv", "w_down", "w_out",
                                   "kv_cache")]
            np.testing.assert_allclose(cp.dense_mla(*args, "absorbed"),
                                       g[f"{name}/dense_absorbed"], atol=1e-6, rtol=0)
            np.testing.assert_allclose(cp.dense_mla(*args, "original"),
                                       g[f"{name}/dense_original"], atol=1e-6, rtol=0)


def test_production_dims_dataflow(golden):
    meta, g = golden
    for name in ("llama2h_n1", "llama2h_n2", "llama2h_n4", "llama2h_n8", "llama2h_n16",
                 "llama_full_s1k_n4", "dsv2_full_s1k_n4"):
        case = next(c for c in meta["cases"] if c["name"] == name)
        arrs = _inputs(case)
        out, smax, ssum = _run_port(case, arrs)
        assert float(np.max(np.abs(out - g[f"{name}/output"]))) <= 2e-3, name
        np.testing.assert_allclose(smax, g[f"{name}/score_max"], atol=2e-3)
        np.testing.assert_allclose(ssum, g[f"{name}/score_sum"], rtol=2e-3)


def test_ffn_reference(golden):
    _, g = golden
    z, w1, w2, w3 = (g[f"ffn/{k}"] for k in ("z", "w1", "w2", "w3"))
    for act in ("silu", "gelu", "relu", "identity"):
        np.testing.assert_allclose(cp.ffn(z, w1, w2, w3, act), g[f"ffn/out_{act}"],
                                   atol=1e-6, rtol=0)


def test_collective_kats(golden):
    meta, g = golden
    for key, info in meta["collectives"].items():
        ins, outs = g[key + "/in"], g[key + "/out"]
        n = ins.shape[0]
        if "/reduce_" in key:
            op = key.split("/reduce_")[1].rsplit("_n", 1)[0]
            tag = cp.tag_for_bytes(int(key.rsplit("_", 1)[1]))
            got = np.stack(cp.ring_reduce(list(ins), op, tag))
            if op == "softmax_merge":
                np.testing.assert_allclose(got, outs, rtol=1e-6, atol=0)
            else:
                assert np.array_equal(got, outs), key
            assert info["dsmem_bytes"] == cp.traffic_reduce(
                ins.shape[1] * int(key.rsplit("_", 1)[1]), n)
        else:
            got = np.stack(cp.ring_gather(list(ins), cp.F32))
            assert np.array_equal(got, outs), key
            for r in range(n):
                assert np.array_equal(cp.canonicalize(got[r], r, n, ins.shape[1]), ins.ravel())
            assert info["dsmem_bytes"] == cp.traffic_gather(ins.shape[1] * 4, n)


def test_known_answers_from_reference_tests():
    """KATs lifted from the reference test suite (values, not code)."""
    # test_collectives.py:61-69
    assert [float(b[0]) for b in cp.ring_reduce([np.array([v], np.float32) for v in (1, 2, 3, 4)],
                                                "sum", cp.F32)] == [10.0] * 4
    assert [float(b[0]) for b in cp.ring_reduce([np.array([5.0], np.float32),
                                                 np.array([-1.0], np.float32)], "max", cp.F32)] \
        == [5.0, 5.0]
    # test_collectives.py:193-205 rotated layout
    bufs = cp.ring_gather([np.array([r + 1], np.float32) for r in range(4)], cp.F32)
    assert bufs[0].tolist() == [1, 4, 3, 2] and bufs[2].tolist() == [3, 2, 1, 4]
    # test_analysis.py:33-41
    assert cp.traffic_reduce(1024, 4) == 8192 and cp.traffic_reduce(256 * 1024, 4) == 2097152
    assert cp.traffic_gather(1024, 4) == 12288 and cp.traffic_gather(1024, 16) == 245760
    # test_dataflows.py:102-107
    assert cp.segments(5, 4) == [(0, 2), (2, 4), (4, 5), (5, 5)]
    assert cp.segments(0, 2) == [(0, 0), (0, 0)]
    # test_dataflows.py:38-46: single key equal to the query
    q = np.array([[1.0, 2.0, 2.0, 1.0]], np.float32)
    v = np.array([[5.0, -3.0, 0.5, 2.0]], np.float32)
    a, m, l = cp.partial_attention(q, q.copy(), v)
    assert m[0] == pytest.approx(10.0 / 2.0) and l[0] == pytest.approx(1.0)
    np.testing.assert_allclose(a, v, atol=1e-6)
    # empty segment -> identity
    a, m, l = cp.partial_attention(np.zeros((3, 4), np.float32), np.zeros((0, 4), np.float32),
                                   np.zeros((0, 4), np.float32))
    assert np.all(a == 0) and np.all(np.isneginf(m)) and np.all(l == 0)
    # softmax merge identity (test_collectives.py:180-185)
    ident = np.array([-np.inf, 0.0], np.float32)
    other = np.array([1.5, 2.0], np.float32)
    np.testing.assert_allclose(cp.merge_stats(ident, other), other)


def test_naive_dual_agrees():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3, 7)).astype(np.float32)
    b = rng.standard_normal((7, 5)).astype(np.float32)
    np.testing.assert_allclose(cp.naive_dot_rows(a, b), a @ b, atol=1e-5)
