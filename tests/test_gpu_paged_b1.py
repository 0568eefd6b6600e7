"""Paged KV cache on the B=1 persistent engine.

The persistent cluster engines read the KV segment of each split_token rank
through a block table (pages of 128 positions, the batched path's
``PagedKVPool`` layout) and append the new row into its page.  Paging changes
only addresses, not arithmetic: the same engine on a shuffled page pool must
give BIT-IDENTICAL logits, tokens and appended rows to the contiguous cache,
which the other persistent tests pin to the CPU oracle."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from oracle import llama_port as lp
from paper_2508_18850_b200.exceptions import DimensionError
from paper_2508_18850_b200.llama import LlamaConfig, LlamaDecoder, random_llama_params

pytestmark = pytest.mark.gpu

SMALL = LlamaConfig(n_layers=3, hidden=512, n_heads=4, head_dim=128, inter=1376, vocab=1000)


def _pair(cfg, prefill, cap, seed, layout="head_major"):
    params = random_llama_params(cfg, seed=seed, prefill=prefill)
    a = LlamaDecoder.from_params(cfg, params, cache_cap=cap)
    b = LlamaDecoder.from_params(cfg, params, cache_cap=cap)
    b.page_kv(shuffle=True, seed=seed, layout=layout)
    return params, a, b


def _same_steps(a, b, pos, tok, steps):
    for s in range(steps):
        for m in (a, b):
            m.set_state(pos, tok)
            m.step()
        la, lb = a.logits(), b.logits()
        assert np.array_equal(la, lb), (s, float(np.max(np.abs(la - lb))))
        assert a.token() == b.token()
        for l in range(a.cfg.n_layers):
            for x, y in zip(a.kv_rows(l, pos), b.kv_rows(l, pos)):
                assert bool((x == y).all()), (s, l)
        tok, pos = a.token(), pos + 1
    a.check()
    b.check()


LAYOUTS = ["head_major", "page_major"]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("engine", ["persistent", "persistent_nodsmem"])
@pytest.mark.parametrize("prefill", [0, 1, 127, 370])
def test_paged_equals_contiguous(engine, prefill, layout):
    cfg = dataclasses.replace(SMALL, engine=engine)
    _, a, b = _pair(cfg, prefill, prefill + 24, seed=11, layout=layout)
    _same_steps(a, b, prefill, 5, steps=20)  # crosses the page edge at 128 / 384


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("cluster", [1, 2, 8])
def test_paged_segments_straddle_pages(cluster, layout):
    """Cluster sizes whose split_token segments start off the 16-row items,
    so ring items span two pages (two bulk copies per source)."""
    cfg = LlamaConfig(n_layers=2, hidden=512, n_heads=8, head_dim=128, inter=1024, vocab=512,
                      cluster=cluster, engine="persistent")
    _, a, b = _pair(cfg, 300, 320, seed=12, layout=layout)
    _same_steps(a, b, 300, 9, steps=6)


def test_paged_matches_oracle_and_graph():
    cfg = dataclasses.replace(SMALL, engine="persistent")
    prefill, steps = 250, 10
    params = random_llama_params(cfg, seed=13, prefill=prefill)
    params["rope_cs"] = lp.rope_table(prefill + steps + 1, cfg.head_dim, cfg.rope_theta)
    caches = [(np.concatenate([l["k_cache"], np.zeros((cfg.n_heads, steps + 1, 128), np.float32)], 1),
               np.concatenate([l["v_cache"], np.zeros((cfg.n_heads, steps + 1, 128), np.float32)], 1))
              for l in params["layers"]]
    m = LlamaDecoder.from_params(cfg, params, cache_cap=prefill + steps + 1)
    m.page_kv()
    ref, tok, pos = [], 4, prefill
    for _ in range(steps):
        _, t = lp.decode_step(params, caches, tok, pos, cfg)
        ref.append(t)
        tok, pos = t, pos + 1
    assert m.generate(first_token=4, pos=prefill, n_tokens=steps, use_graph=True) == ref


def test_unreserved_page_is_flagged_then_served():
    cfg = dataclasses.replace(SMALL, engine="persistent")
    params = random_llama_params(cfg, seed=14, prefill=127)
    a = LlamaDecoder.from_params(cfg, params, cache_cap=300)
    b = LlamaDecoder.from_params(cfg, params, cache_cap=300)
    pool = b.page_kv(reserve=128)  # page 0 only
    for m in (a, b):
        m.set_state(127, 3)
        m.step()  # row 127: page 0
    a.check()
    b.check()
    assert np.array_equal(a.logits(), b.logits())
    b.set_state(128, a.token())
    b.step()  # row 128 lands on an unreserved page: nothing done, flagged
    with pytest.raises(DimensionError):
        b.check()
    pool.reserve(0, 129)
    _same_steps(a, b, 128, a.token(), steps=3)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_paged_llama_width_long_context(layout):
    """Llama2-7B width (2 layers), 4K context, cluster 4: bit-identical to the
    contiguous cache (the contiguous engine is oracle-tested at this width)."""
    cfg = LlamaConfig(n_layers=2, hidden=4096, n_heads=32, head_dim=128, inter=11008, vocab=32000,
                      engine="persistent")
    a = LlamaDecoder.random(cfg, cache_cap=4100, seed=21)
    b = LlamaDecoder.random(cfg, cache_cap=4100, seed=21)
    b.page_kv(seed=3, layout=layout)
    _same_steps(a, b, 4093, 17, steps=3)


def test_paged_rejects_flat_engine_and_oversized_segments():
    cfg = dataclasses.replace(SMALL, engine="persistent_flat")
    m = LlamaDecoder.from_params(cfg, random_llama_params(cfg, seed=1, prefill=4), cache_cap=16)
    with pytest.raises(DimensionError):
        m.page_kv()
    m2 = LlamaDecoder.from_params(SMALL, random_llama_params(SMALL, seed=1, prefill=4), cache_cap=16)
    m2.page_kv()
    with pytest.raises(DimensionError):  # already paged
        m2.page_kv()
    # cluster 1 keeps a whole 32K-position sequence on one CTA: more pages than the producer holds
    cfg1 = LlamaConfig(n_layers=1, hidden=512, n_heads=4, head_dim=128, inter=1024, vocab=512, cluster=1)
    m1 = LlamaDecoder.random(cfg1, cache_cap=32768, seed=2)
    m1.page_kv()
    m1.set_state(5, 1)
    with pytest.raises(DimensionError):
        m1.step()


def test_paged_graph_replay_with_incremental_reserve():
    """The INTEGRATION.md loop: the captured graph keeps the table pointer and
    sees pages reserved between replays (a new page every 128 positions)."""
    cfg = dataclasses.replace(SMALL, engine="persistent")
    params = random_llama_params(cfg, seed=15, prefill=120)
    a = LlamaDecoder.from_params(cfg, params, cache_cap=400)
    b = LlamaDecoder.from_params(cfg, params, cache_cap=400)
    pool = b.page_kv(reserve=121)
    ref = a.generate(first_token=6, pos=120, n_tokens=20, use_graph=True)
    b.set_state(120, 6)
    b.step()
    b.set_state(120, 6)
    b.capture()
    got, pos = [], 120
    for _ in range(20):
        pool.reserve(0, pos + 1)
        b.replay()
        got.append(b.token())
        pos += 1
    b.check()
    assert got == ref
    assert len(pool.pages[0]) == 2  # positions 0..139: pages 0 and 1
