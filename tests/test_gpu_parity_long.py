"""GPU parity at the configurations bench.py times (BASELINE configs[0]/[1]/[4]).

The benchmark runs Llama2-7B widths (D=4096, 32x128 heads, F=11008,
V=32000), 32 layers, contexts 1K-16K, and the batch-16 stack at 1K/4K.  These
tests run the same code paths at those sizes against the CPU oracle:

* the drop-in ``run_fused_mha_decode`` (all 32 heads, N=4, fp16) at
  S = 2047 / 4096 / 8192 / 16383 against the dense fp32 oracle
  (reference ``oracle.py:30-52``), i.e. per-CTA KV segments of 512-4096 rows;
* the B=1 engine at full width, 2 layers, prefill 4095 and 16383 (RoPE at
  positions > 1K, segment lengths of the benched contexts);
* the whole 32-layer engine at 1K, generated and checked one layer at a time
  (layer-major: each layer processes the three teacher-forced tokens before
  the next layer is drawn, so host memory holds one fp32 layer);
* the batch-16 stack at Llama width with ragged contexts up to 4K.

Tolerances (north star): logits / hidden states max-abs <= 2e-2 and max-rel
(max|err| / max|ref|) <= 1e-2 against the fp32-accumulated CPU reference;
greedy tokens equal, unconditionally, with the oracle's top-2 margins printed.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import paper_2508_18850_b200 as cfb
from oracle import clusterdec_port as cp
from oracle import llama_port as lp
from paper_2508_18850_b200.llama import (LlamaConfig, LlamaDecoder, random_llama_globals,
                                         random_llama_layer)

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 1e-2


def _err(got, ref):
    a = float(np.max(np.abs(got - ref)))
    return a, a / max(float(np.max(np.abs(ref))), 1e-30)


@pytest.mark.parametrize("S", [2047, 4096, 8192, 16383])
def test_split_token_llama_module_long_context(S):
    """config #1's attention module (all heads) at the benched context lengths."""
    dims = cfb.ModelDims(1, 4096, 32, 128, S, dtype_bytes=2)
    sc = cfb.random_mha_scenario(dims, n_blocks=4, seed=100 + S)
    res = cfb.run_fused_mha_decode(sc)
    ref = cp.dense_mha(sc.hidden, sc.w_qkv, sc.w_out, sc.k_cache, sc.v_cache)
    a, r = _err(res.output, ref)
    print(f"S={S}: max-abs {a:.3e} max-rel {r:.3e}")
    assert a <= ATOL and r <= RTOL, (a, r)
    # the cluster-partitioned restatement with the reference's f16 storage
    # rounding (simcore.py:45-110): output and stats agree tightly
    o32, sm, ss = cp.split_token({k: getattr(sc, k) for k in
                                  ("hidden", "w_qkv", "w_out", "k_cache", "v_cache")},
                                 4, 2, head_accum="f32")
    assert float(np.max(np.abs(res.output - o32))) <= 2e-3
    np.testing.assert_allclose(res.score_max, sm, atol=2e-3)
    np.testing.assert_allclose(res.score_sum, ss, rtol=2e-3)
    # vs the dense fp32 statistics: score_sum is an fp16 store (f16 mode) after
    # log2(N) fp16-rounded rescale+add rounds, i.e. a few fp16 ulps (2^-10)
    m, l = cp.dense_mha_stats(sc.hidden, sc.w_qkv, sc.k_cache)
    np.testing.assert_allclose(res.score_max, m, atol=2e-3)
    np.testing.assert_allclose(res.score_sum, l, rtol=4 * 2.0 ** -10)
    assert cfb.reconcile_traffic("split_token", res, sc.dims).reconciled


def _teacher_forced_layer_major(cfg, prefill, tokens, seed, engines=("persistent",)):
    """Run the oracle layer by layer over all teacher-forced tokens while the
    engines are packed from the same layers; returns (engines, oracle logits)."""
    T = len(tokens)
    cap = prefill + T + 1
    g = random_llama_globals(cfg, seed)
    cs = lp.rope_table(cap, cfg.head_dim, cfg.rope_theta)
    x = g["embed"][tokens].astype(np.float32)  # (T, D): residual stream per step

    def layers():
        nonlocal x
        for l in range(cfg.n_layers):
            L = random_llama_layer(cfg, seed, l, prefill)
            kc = np.zeros((cfg.n_heads, cap, cfg.head_dim), np.float32)
            vc = np.zeros_like(kc)
            kc[:, :prefill], vc[:, :prefill] = L["k_cache"], L["v_cache"]
            for t in range(T):  # token t sits at position prefill + t
                xt = x[t:t + 1]
                h = lp.rmsnorm_f16(xt, L["attn_norm"], cfg.eps)
                xt = xt + lp.attention_module(h, L["w_qkv"], L["w_out"], kc, vc, prefill + t,
                                              cfg.cluster, cs)
                xt = xt + lp.ffn_block(xt, L["ffn_norm"], L["w1"], L["w2"], L["w3"], cfg.eps)
                x[t] = xt[0]
            yield L
            del L, kc, vc

    ms = [LlamaDecoder(dataclasses.replace(cfg, engine=e), cap) for e in engines]

    def pack_all():
        for L in layers():
            for m in ms:
                m.layers.append(m._pack_layer(L))
            yield L

    for _ in pack_all():
        pass
    for m in ms:
        m.adopt_globals(g)
    hf = lp.rmsnorm_f16(x, g["final_norm"], cfg.eps)
    logits = (hf @ g["lm_head"].T).astype(np.float32)
    return ms, logits


def _check_engine(m, tokens, prefill, ref_logits):
    margins = []
    for t, tok in enumerate(tokens):
        m.set_state(prefill + t, tok)
        m.step()
        got = m.logits()
        a, r = _err(got, ref_logits[t])
        top2 = np.sort(ref_logits[t])[-2:]
        margins.append(float(top2[1] - top2[0]))
        print(f"step {t}: max-abs {a:.3e} max-rel {r:.3e} top-2 margin {margins[-1]:.4f}")
        assert a <= ATOL and r <= RTOL, (t, a, r)
        assert m.token() == int(np.argmax(ref_logits[t])), (t, margins[-1])
    return margins


@pytest.mark.parametrize("prefill", [4095, 16383])
def test_engine_full_width_long_prefill(prefill):
    """Llama2-7B widths, 2 layers, the benched 4K / 16K contexts (both engines)."""
    cfg = LlamaConfig(n_layers=2)
    tokens = [7, 3051, 29999]
    ms, ref = _teacher_forced_layer_major(cfg, prefill, tokens, seed=40 + prefill % 7,
                                          engines=("persistent", "layered"))
    for m in ms:
        _check_engine(m, tokens, prefill, ref)


def test_engine_32_layers_1k():
    """The whole benched model (32 layers) at the 1K context, 3 teacher-forced
    greedy steps, graph replay included."""
    import torch
    cfg = LlamaConfig()
    tokens = [7, 3051, 29999]
    prefill = 1024
    (m,), ref = _teacher_forced_layer_major(cfg, prefill, tokens, seed=77)
    _check_engine(m, tokens, prefill, ref)
    # the CUDA-graph replay path (what bench.py times) gives the same tokens
    got = []
    m.set_state(prefill, tokens[0])
    m.capture()
    for t, tok in enumerate(tokens):
        m.set_state(prefill + t, tok)
        m.replay()
        got.append(m.token())
    torch.cuda.synchronize()
    assert got == [int(np.argmax(r)) for r in ref]


def test_batched_llama_width_ragged_4k():
    """The batch-16 stack (tcgen05 projections) at Llama2-7B widths, 2 layers,
    16 independent sequences with ragged contexts up to 4K, 2 greedy steps:
    logits within 2e-2 abs / 1e-2 rel of the per-sequence oracle, tokens equal."""
    import torch
    from paper_2508_18850_b200.batched import BatchedLlama
    from paper_2508_18850_b200.llama import rope_table
    cfg = LlamaConfig(n_layers=2)
    seed = 21
    rng = np.random.default_rng(seed)
    S = [4096, 1, 127, 128, 129, 1000, 1023, 1024, 1025, 2047, 2048, 3000, 3500, 4000, 4095, 512]
    steps = 2
    cap = max(S) + steps + 2
    layers = [random_llama_layer(cfg, seed, l) for l in range(cfg.n_layers)]
    g = random_llama_globals(cfg, seed)
    caches = [[(lp.f16(rng.standard_normal((cfg.n_heads, s, 128), dtype=np.float32)),
                lp.f16(rng.standard_normal((cfg.n_heads, s, 128), dtype=np.float32))) for s in S]
              for _ in range(cfg.n_layers)]
    m = BatchedLlama.from_params(cfg, layers, caches, cache_cap=cap)
    m.set_head(g["embed"], g["final_norm"], g["lm_head"])
    toks = [int(t) for t in rng.integers(0, cfg.vocab, 16)]
    m.tokens.copy_(torch.tensor(toks, dtype=torch.int32))
    m.set_positions(S)
    oparams = dict(g, layers=layers, rope_cs=rope_table(cap, 128, cfg.rope_theta))
    ocache = []
    for n in range(16):
        per = []
        for l in range(cfg.n_layers):
            kc = np.zeros((cfg.n_heads, S[n] + steps + 1, 128), np.float32)
            vc = np.zeros_like(kc)
            kc[:, :S[n]], vc[:, :S[n]] = caches[l][n]
            per.append((kc, vc))
        ocache.append(per)
    del caches
    worst = 0.0
    for step in range(steps):
        m.decode_step(logits=True)
        torch.cuda.synchronize()
        got = m.tokens.cpu().tolist()
        glog = m.logits.cpu().numpy()
        for n in range(16):
            ologits, otok = lp.decode_step(oparams, ocache[n], toks[n], S[n] + step, cfg)
            a, r = _err(glog[n], ologits)
            worst = max(worst, a)
            top2 = np.sort(ologits)[-2:]
            assert a <= ATOL and r <= RTOL, (step, n, a, r)
            assert got[n] == otok, (step, n, got[n], otok, float(top2[1] - top2[0]))
            toks[n] = otok
        m.tokens.copy_(torch.tensor(toks, dtype=torch.int32))
    print(f"batch-16 Llama width: worst logits max-abs {worst:.3e}")
