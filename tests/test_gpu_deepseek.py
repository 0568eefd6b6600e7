"""GPU parity of the DeepSeek-V2-Lite-shaped decoder block (fused_mla with
RMSNorm prologue -> fused MoE with residual + RMSNorm + router + experts)
against the CPU restatement ``oracle/deepseek_port.block``.

Tolerance: north-star max-abs 2e-2 / max-rel 1e-2 on the block output (the
residual stream); expert selection equal whenever the oracle's top-k margin
is not a near-tie.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import clusterdec_port as cp
from oracle import deepseek_port as dp
from oracle.llama_port import f16
from paper_2508_18850_b200.deepseek import DeepSeekBlock, DeepSeekDims

pytestmark = pytest.mark.gpu

MLA_KEYS = ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _case(dims: DeepSeekDims, S, B, seed):
    rng = np.random.default_rng(seed)
    mla = cp.gen_mla(B, dims.hidden, dims.n_heads, dims.head_dim, S, dims.kv_rank, 2, seed=seed)
    mla = {k: mla[k] for k in MLA_KEYS}
    moe_w = dp.gen_moe(dims.hidden, dims.n_experts, dims.inter, dims.n_shared, seed=seed)
    ga = f16(1 + 0.1 * rng.standard_normal(dims.hidden))
    gf = f16(1 + 0.1 * rng.standard_normal(dims.hidden))
    x = rng.standard_normal((B, dims.hidden)).astype(np.float32)
    return mla, moe_w, ga, gf, x


@pytest.mark.parametrize("B,cluster,S", [(1, 2, 40), (2, 4, 33), (3, 1, 7), (1, 4, 0)])
def test_block_small_dims(B, cluster, S):
    dims = DeepSeekDims(hidden=256, n_heads=4, head_dim=32, kv_rank=64, n_experts=8, top_k=2,
                        inter=32, n_shared=1, cluster=cluster)
    mla, moe_w, ga, gf, x = _case(dims, S, B, seed=S + B)
    blk = DeepSeekBlock.from_arrays(dims, mla, moe_w, ga, gf, batch=B)
    out, idx = blk.run(x)
    ref, info = dp.block(x, mla, ga, gf, moe_w, dims.top_k, cluster, dims.eps)
    if np.all(info["margin"] > 1e-4):
        assert np.array_equal(np.sort(idx, 1), np.sort(info["idx"], 1))
    assert float(np.max(np.abs(out - ref))) <= 2e-2 and _rel(out, ref) <= 1e-2


@pytest.mark.parametrize("S,engine", [(1, False), (300, False), (0, True), (1, True), (300, True),
                                      (2000, True)])
def test_block_lite_dims(S, engine):
    """engine=True: the head-batched MLA engine (csrc/mla_engine.cu);
    False: the reference-dataflow fused_mla kernel."""
    dims = DeepSeekDims()  # MLA preset dims + DeepSeek-V2-Lite MoE
    mla, moe_w, ga, gf, x = _case(dims, S, 1, seed=7)
    blk = DeepSeekBlock.from_arrays(dims, mla, moe_w, ga, gf, use_engine=engine)
    assert (blk.engine is not None) == engine
    out, idx = blk.run(x)
    ref, info = dp.block(x, mla, ga, gf, moe_w, dims.top_k, dims.cluster, dims.eps)
    assert info["margin"][0] > 1e-4
    assert np.array_equal(np.sort(idx, 1), np.sort(info["idx"], 1))
    assert float(np.max(np.abs(out - ref))) <= 2e-2 and _rel(out, ref) <= 1e-2
    # second launch on the updated stream reuses (re-zeroed) workspaces
    out2, _ = blk.run(out)
    ref2, _ = dp.block(out, mla, ga, gf, moe_w, dims.top_k, dims.cluster, dims.eps)
    assert float(np.max(np.abs(out2 - ref2))) <= 2e-2 and _rel(out2, ref2) <= 1e-2


def test_mla_engine_attention_half_matches_dense_oracle():
    """The engine's attention half alone (head sum in the fixed-point
    accumulator) vs the dense fp32 MLA oracle (oracle.py:55-93 absorbed)."""
    import torch
    from oracle.llama_port import rmsnorm_f16
    dims = DeepSeekDims()
    for S in (5, 700, 5000):
        mla, moe_w, ga, gf, x = _case(dims, S, 1, seed=S)
        blk = DeepSeekBlock.from_arrays(dims, mla, moe_w, ga, gf)
        r = torch.from_numpy(x).cuda()
        blk.launch_attention(r, pdl=False)
        torch.cuda.synchronize()
        got = blk.accum_attn.cpu().numpy().astype(np.float64) * 2.0 ** -32
        blk.accum_attn.zero_()
        h = rmsnorm_f16(x, ga, dims.eps)
        ref = cp.dense_mla(h, *(mla[k] for k in ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")))
        assert float(np.max(np.abs(got - ref))) <= 2e-2 and _rel(got, ref) <= 1e-2, S
