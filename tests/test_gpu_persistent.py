"""The persistent whole-step engine (csrc/decode_step.cu) against the CPU
oracle and against the layered engine: same packed weights, same greedy
tokens; logits within the north-star tolerance (2e-2 abs / 1e-2 rel)."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from oracle import llama_port as lp
from paper_2508_18850_b200.llama import LlamaConfig, LlamaDecoder, random_llama_params

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _run(cfg, prefill, steps, seed):
    params = random_llama_params(cfg, seed=seed, prefill=prefill)
    params["rope_cs"] = lp.rope_table(prefill + steps + 1, cfg.head_dim, cfg.rope_theta)
    caches = [(np.concatenate([l["k_cache"], np.zeros((cfg.n_heads, steps + 1, cfg.head_dim),
                                                      np.float32)], 1),
               np.concatenate([l["v_cache"], np.zeros((cfg.n_heads, steps + 1, cfg.head_dim),
                                                      np.float32)], 1)) for l in params["layers"]]
    m = LlamaDecoder.from_params(cfg, params, cache_cap=prefill + steps + 1)
    tok, pos = 7, prefill
    for s in range(steps):
        ref_logits, ref_tok = lp.decode_step(params, caches, tok, pos, cfg)
        m.set_state(pos, tok)
        m.step()
        got = m.logits()
        err = float(np.max(np.abs(got - ref_logits)))
        assert err <= 2e-2 and _rel(got, ref_logits) <= 1e-2, (s, err)
        assert m.token() == ref_tok, (s, m.token(), ref_tok)
        # the appended K/V rows equal the oracle's (fp16 values)
        for l, (kc, vc) in enumerate(caches):
            gk = m.layers[l]["k_cache"][:, pos].float().cpu().numpy()
            assert float(np.max(np.abs(gk - kc[:, pos]))) <= 2e-2, (s, l)
        tok, pos = ref_tok, pos + 1
    return m


ENGINES = ["persistent", "persistent_flat", "persistent_nodsmem"]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("prefill", [0, 1, 3, 37, 300])
def test_persistent_small(prefill, engine):
    cfg = LlamaConfig(n_layers=3, hidden=512, n_heads=4, head_dim=128, inter=1376, vocab=1000,
                      engine=engine)
    _run(cfg, prefill, steps=4, seed=1)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cluster", [1, 2, 8])
def test_persistent_reads_any_split_token_layout(cluster, engine):
    cfg = LlamaConfig(n_layers=2, hidden=512, n_heads=8, head_dim=128, inter=1024, vocab=512,
                      cluster=cluster, engine=engine)
    _run(cfg, 100, steps=3, seed=2)


@pytest.mark.parametrize("engine", ENGINES)
def test_persistent_matches_layered_tokens_graph(engine):
    cfg = LlamaConfig(n_layers=2, hidden=512, n_heads=4, head_dim=128, inter=1376, vocab=1000,
                      engine="layered")
    params = random_llama_params(cfg, seed=5, prefill=20)
    a = LlamaDecoder.from_params(cfg, params, cache_cap=64)
    b = LlamaDecoder.from_params(dataclasses.replace(cfg, engine=engine), params, cache_cap=64)
    assert b.launches_per_step == 1
    ta = a.generate(first_token=3, pos=20, n_tokens=8, use_graph=True)
    tb = b.generate(first_token=3, pos=20, n_tokens=8, use_graph=True)
    assert ta == tb


@pytest.mark.parametrize("engine", ENGINES)
def test_persistent_full_cache_is_flagged(engine):
    cfg = LlamaConfig(n_layers=1, hidden=512, n_heads=4, head_dim=128, inter=1376, vocab=1000,
                      engine=engine)
    m = LlamaDecoder.from_params(cfg, random_llama_params(cfg, seed=3, prefill=8), cache_cap=10)
    m.set_state(9, 1)
    m.step()  # pos 9 -> fills row 9 (cap 10)
    m.check()
    m.step()  # pos 10 == cap: skipped, flagged
    from paper_2508_18850_b200.exceptions import DimensionError
    with pytest.raises(DimensionError):
        m.check()


@pytest.mark.parametrize("engine", ENGINES)
def test_persistent_trace_stamps_monotone(engine):
    cfg = LlamaConfig(n_layers=2, hidden=512, n_heads=4, head_dim=128, inter=1376, vocab=1000,
                      engine=engine)
    m = LlamaDecoder.from_params(cfg, random_llama_params(cfg, seed=4, prefill=16), cache_cap=32)
    tr = m.set_trace(True)
    m.set_state(16, 2)
    m.step()
    m.stream.synchronize()
    t = tr.cpu().numpy()
    assert (t > 0).all()
    assert (np.diff(t, axis=2) >= 0).all()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_persistent_tp_shard_cluster(world):
    """One rank's shard of the fused tensor-parallel path at Llama2-7B width
    with the cluster size `fused_local_config` picks for it (TP2: 4, TP4: 8,
    TP8: 16 - non-portable), against the oracle on the shard's dims."""
    from paper_2508_18850_b200.tp_fused import fused_local_config
    full = LlamaConfig(n_layers=2, hidden=4096, n_heads=32, head_dim=128, inter=11008, vocab=32000)
    cfg = fused_local_config(full, world)
    assert cfg.cluster == {2: 4, 4: 8, 8: 16}[world]
    _run(cfg, 700, steps=2, seed=10 + world)
