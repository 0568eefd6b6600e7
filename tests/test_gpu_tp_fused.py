"""Fused tensor parallel (in-kernel all-reduce over peer memory, one launch
per token per rank) on one B200: all ranks in one process, each on its own
stream and a 1/T share of the SMs (tp_fused.emulated_ranks), the same kernel
code and cross-rank protocol a multi-GPU run uses.  Checked against the CPU
oracle of the UNSHARDED model (north-star tolerance 2e-2 abs / 1e-2 rel,
greedy tokens equal) and for run-to-run bit-identity (the fixed-point sums
make the result independent of which rank arrives first)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import llama_port as lp
from paper_2508_18850_b200.llama import LlamaConfig, random_llama_params
from paper_2508_18850_b200.tp_fused import emulated_ranks

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _oracle_caches(params, cfg, steps):
    return [(np.concatenate([l["k_cache"], np.zeros((cfg.n_heads, steps + 1, cfg.head_dim), np.float32)], 1),
             np.concatenate([l["v_cache"], np.zeros((cfg.n_heads, steps + 1, cfg.head_dim), np.float32)], 1))
            for l in params["layers"]]


def _run(cfg, world, prefill, steps, seed, graph=False, nvls=False):
    params = random_llama_params(cfg, seed=seed, prefill=prefill)
    params["rope_cs"] = lp.rope_table(prefill + steps + 1, cfg.head_dim, cfg.rope_theta)
    caches = _oracle_caches(params, cfg, steps)
    tp = emulated_ranks(cfg, world, prefill + steps + 1, params=params, timeout_s=5.0, nvls=nvls)
    tok, pos = 7, prefill
    seen = []
    for s in range(steps):
        ref_logits, ref_tok = lp.decode_step(params, caches, tok, pos, cfg)
        tp.set_state(pos, tok)
        if graph and s == 0:
            tp.step()
            tp.set_state(pos, tok)
            tp.capture()
        tp.replay() if graph else tp.step()
        tp.check()
        got = tp.logits()
        err = float(np.max(np.abs(got - ref_logits)))
        assert err <= 2e-2 and _rel(got, ref_logits) <= 1e-2, (s, err)
        toks = tp.tokens()
        assert toks == [ref_tok] * world, (s, toks, ref_tok)
        seen.append(got)
        tok, pos = ref_tok, pos + 1
    return tp, seen


SMALL = dict(n_layers=3, hidden=512, n_heads=8, head_dim=128, inter=1408, vocab=1024)


@pytest.mark.parametrize("engine", ["persistent", "persistent_flat"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("prefill", [0, 37, 300])
def test_fused_tp_small_matches_unsharded_oracle(world, prefill, engine):
    cfg = LlamaConfig(**SMALL, engine=engine)
    _run(cfg, world, prefill, steps=3, seed=5)


@pytest.mark.parametrize("world", [2, 4])
def test_fused_tp_bit_identical_runs_and_graph(world):
    cfg = LlamaConfig(**SMALL)
    _, a = _run(cfg, world, 64, steps=2, seed=9)
    _, b = _run(cfg, world, 64, steps=2, seed=9, graph=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_tp_llama_width(world):
    """Llama2-7B widths (D 4096, 32 heads, F 11008, V 32000), 2 layers: head
    shards of 16 / 8 / 4 heads per rank."""
    cfg = LlamaConfig(n_layers=2)
    _run(cfg, world, 300, steps=2, seed=3)


def _need_nvls():
    from paper_2508_18850_b200.tp_fused import nvls_usable
    if not nvls_usable(0):
        pytest.skip("no usable NVLS multicast on this GPU (cuMulticastCreate refused)")


@pytest.mark.parametrize("world", [2, 4])
def test_fused_tp_nvls_sums_match_oracle_and_peer_path(world):
    """The sums on an NVLS multicast buffer (multimem.red.add.u64 on the
    multicast mapping, csrc/nvls.cu; emulated ranks share the one-member
    object's copy): oracle parity, and bit-identical to the peer-memory
    pushes (fixed-point sums are order-free)."""
    _need_nvls()
    cfg = LlamaConfig(**SMALL)
    _, a = _run(cfg, world, 64, steps=3, seed=11)
    tp, b = _run(cfg, world, 64, steps=3, seed=11, nvls=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    _, c = _run(cfg, world, 64, steps=3, seed=11, graph=True, nvls=True)
    for x, y in zip(a, c):
        assert np.array_equal(x, y)


def test_nvls_setup_path_single_member():
    """The multicast-object setup a multi-GPU group runs (create, add device,
    bind: a zeroed physical copy with unicast + multicast mappings), with one
    member; the reductions through it are checked by the test above."""
    import torch
    _need_nvls()
    from paper_2508_18850_b200.tp_fused import NvlsSums
    s = NvlsSums(4096, torch.cuda.current_device())
    assert s.uc.value and s.mc.value and s.uc.value != s.mc.value
    assert int(s._L.cfb_nvls_size(s.h)) >= 6 * 4096 * 8
    del s
    torch.cuda.synchronize()
