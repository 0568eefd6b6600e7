"""Greedy decode of a whole DeepSeek-shaped model (embedding -> 3 blocks of
head-batched MLA engine + fused MoE -> final RMSNorm + LM head + argmax), one
CUDA graph per step, against the CPU restatement (oracle/deepseek_port.block
per layer + the LM head of oracle/llama_port), teacher-forced.  Tolerance:
north-star 2e-2 abs / 1e-2 rel on the logits; greedy tokens equal
unconditionally (the oracle's top-2 margin is printed)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import clusterdec_port as cp
from oracle import deepseek_port as dp
from oracle.llama_port import f16, rmsnorm_f16
from paper_2508_18850_b200.deepseek import DeepSeekDims
from paper_2508_18850_b200.deepseek_model import DeepSeekDecoder, DeepSeekModelDims

pytestmark = pytest.mark.gpu
MLA_KEYS = ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")


@pytest.mark.parametrize("S", [37, 700])
def test_deepseek_model_greedy_teacher_forced(S):
    bd = DeepSeekDims(hidden=512, n_heads=4, head_dim=64, kv_rank=512, n_experts=8, top_k=2, inter=64,
                      n_shared=1)
    md = DeepSeekModelDims(block=bd, n_layers=3, vocab=512)
    rng = np.random.default_rng(S)
    layers = []
    for l in range(md.n_layers):
        mla = cp.gen_mla(1, bd.hidden, bd.n_heads, bd.head_dim, S, bd.kv_rank, 2, seed=100 * S + l)
        mla = {k: mla[k] for k in MLA_KEYS}
        moe_w = dp.gen_moe(bd.hidden, bd.n_experts, bd.inter, bd.n_shared, seed=100 * S + l)
        ga = f16(1 + 0.1 * rng.standard_normal(bd.hidden))
        gf = f16(1 + 0.1 * rng.standard_normal(bd.hidden))
        layers.append((mla, moe_w, ga, gf))
    embed = f16(rng.standard_normal((md.vocab, bd.hidden)))
    fnorm = f16(1 + 0.1 * rng.standard_normal(bd.hidden))
    lm = f16(rng.standard_normal((md.vocab, bd.hidden)) * bd.hidden ** -0.5)
    m = DeepSeekDecoder.from_arrays(md, layers, embed, fnorm, lm)
    tok = 3
    for step in range(3):
        x = embed[tok:tok + 1].astype(np.float32)
        for (mla, moe_w, ga, gf) in layers:
            x, _ = dp.block(x, mla, ga, gf, moe_w, bd.top_k, bd.cluster, bd.eps)
        ologits = (rmsnorm_f16(x, fnorm, bd.eps) @ lm.T)[0]
        otok = int(np.argmax(ologits))
        if step == 2:  # the captured CUDA graph of the step produces the same token
            m.capture()
            m.set_token(tok)
            m.replay()
            assert m.token() == otok
        m.set_token(tok)
        m.step(logits=True)
        got = m.logits()
        err = float(np.max(np.abs(got - ologits)))
        top2 = np.sort(ologits)[-2:]
        print(f"S={S} step {step}: max-abs {err:.3e} top-2 margin {top2[1] - top2[0]:.4f}")
        assert err <= 2e-2 and err / float(np.max(np.abs(ologits))) <= 1e-2, (step, err)
        assert m.token() == otok, (step, m.token(), otok)
        tok = otok
