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
