"""Tensor-parallel decode on the GPU.

* TP=2 emulated on one device: two rank engines (head / FFN-column / vocab
  shards, rank 0 adds the residual) driven through the real ``tp_step``
  schedule, with the three collectives done by device-side sums/max between
  the ranks' buffers; tokens must equal the unsharded engine's, logits match.
* The NCCL path: a world-size-1 NCCL process group with the collectives
  forced on, captured in a CUDA graph together with the kernels.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from paper_2508_18850_b200.llama import LlamaConfig, LlamaDecoder, random_llama_params
from paper_2508_18850_b200.tp import TPLlamaDecoder, tp_step

pytestmark = pytest.mark.gpu

CFG = LlamaConfig(n_layers=2, hidden=512, n_heads=4, head_dim=128, inter=1408, vocab=1024, cluster=4)


class PairOps:
    """Lock-step ops over the rank engines of one emulated TP group."""

    def __init__(self, decs):
        self.decs = decs

    def _each(self, name, *a):
        for d in self.decs:
            getattr(d.ops, name)(*a)

    def embed(self):
        self._each("embed")

    def attn(self, l):
        self._each("attn", l)

    def ffn(self, l):
        self._each("ffn", l)

    def head(self):
        self._each("head")

    def token(self):
        self._each("token")

    def _reduce(self, attr, fn):
        torch.cuda.synchronize()
        ts = [getattr(d, attr) for d in self.decs]
        r = ts[0].clone()
        for t in ts[1:]:
            r = fn(r, t)
        for t in ts:
            t.copy_(r)
        torch.cuda.synchronize()

    def allreduce_heads(self):
        self._reduce("accum", torch.add)

    def allreduce_resid(self):
        self._reduce("resid", torch.add)

    def allreduce_argmax(self):
        self._reduce("argkey", torch.maximum)


@pytest.mark.parametrize("world", [2, 4])
def test_tp_emulated_matches_single_engine(world):
    params = random_llama_params(CFG, seed=11, prefill=30)
    ref = LlamaDecoder.from_params(CFG, params, cache_cap=64)
    ref.set_state(30, 7)
    decs = [TPLlamaDecoder(CFG, r, world, 64, params=params) for r in range(world)]
    for d in decs:
        d.set_state(30, 7)
    ops = PairOps(decs)
    for s in range(4):
        ref.step()
        tref = ref.token()
        lref = ref.logits()
        tp_step(ops, CFG.n_layers)
        toks = [d.token() for d in decs]
        assert toks == [tref] * world, (s, toks, tref)
        local = np.concatenate([d.logits_local() for d in decs])
        assert float(np.max(np.abs(local - lref))) <= 2e-2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp_nccl_graph_world1():
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        params = random_llama_params(CFG, seed=12, prefill=20)
        ref = LlamaDecoder.from_params(CFG, params, cache_cap=64)
        want = ref.generate(first_token=3, pos=20, n_tokens=5, use_graph=False)
        d = TPLlamaDecoder(CFG, 0, 1, 64, params=params, force_collectives=True)
        d.set_state(20, 3)
        d.step()  # configure kernels outside capture
        torch.cuda.synchronize()
        d.set_state(20, 3)
        d.capture()
        got = []
        for _ in range(5):
            d.replay()
            got.append(d.token())
        assert got == want
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S", [(2, 300), (4, 300), (4, 10000)])  # 10000: 148 attention partials
def test_tp_deepseek_block_emulated(world, S):
    """TP DeepSeek block on one device: per-rank MLA engine on its heads
    (world 4: one head per rank, the NH = 1 engine path) -> device int64 SUM of
    the fixed-point attention partials -> per-rank MoE on its expert-row shard
    (CFB_PARTIAL on ranks > 0) -> device SUM == the unsharded block."""
    import torch
    from oracle import clusterdec_port as cp
    from oracle import deepseek_port as dp
    from paper_2508_18850_b200.deepseek import DeepSeekBlock, DeepSeekDims
    from paper_2508_18850_b200.tp import TPDeepSeekBlock
    dims = DeepSeekDims(hidden=512, n_heads=4, head_dim=64, kv_rank=512, n_experts=8, top_k=2, inter=128,
                        n_shared=1)
    mla = cp.gen_mla(1, dims.hidden, dims.n_heads, dims.head_dim, S, dims.kv_rank, seed=4)
    mla = {k: mla[k] for k in ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")}
    moe_w = dp.gen_moe(dims.hidden, dims.n_experts, dims.inter, dims.n_shared, seed=6)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, dims.hidden)).astype(np.float32)
    g1 = dp.f16(1.0 + 0.1 * rng.standard_normal(dims.hidden))
    g2 = dp.f16(1.0 + 0.1 * rng.standard_normal(dims.hidden))
    full = DeepSeekBlock.from_arrays(dims, mla, moe_w, g1, g2)
    assert full.engine is not None
    want, want_idx = full.run(x)
    ranks = [TPDeepSeekBlock.from_arrays(dims, mla, moe_w, g1, g2, r, world) for r in range(world)]
    assert all(t.block.engine is not None for t in ranks)
    rs = [torch.from_numpy(x).cuda() for _ in range(world)]
    for t, r in zip(ranks, rs):
        t.launch_attention(r)
    acc = sum(t.block.accum_attn for t in ranks)       # int64: exact, as the NCCL SUM
    for t in ranks:
        t.block.accum_attn.copy_(acc)
    for t, r in zip(ranks, rs):
        t.launch_moe(r)
    got = sum(rs).cpu().numpy()
    torch.cuda.synchronize()
    for t in ranks:
        assert np.array_equal(t.block.ws.route_idx.cpu().numpy().astype(np.int64), want_idx)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=2e-5)
    # and against the CPU oracle block at the north-star tolerance
    ref, _ = dp.block(x, mla, g1, g2, moe_w, dims.top_k, dims.cluster, dims.eps, dims.routed_scale)
    err = float(np.max(np.abs(got - ref)))
    assert err <= 2e-2 and err / float(np.max(np.abs(ref))) <= 1e-2, err
