"""Tensor-parallel schedule on CPU: two gloo ranks run ``tp.tp_step`` (the
exact schedule the GPU driver runs: shard -> attention half -> int64 SUM of
the fixed-point head sum -> FFN half (residual on rank 0) -> fp32 SUM ->
vocab-sharded argmax -> int64 MAX of packed keys) with the numpy oracle as
the per-rank compute, and must reproduce the single-process oracle step."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import llama_port as lp
from paper_2508_18850_b200.llama import LlamaConfig, random_llama_params, rope_table
from paper_2508_18850_b200.tp import (check_tp, local_config, pack_argmax_key, shard_params,
                                      tp_step, unpack_argmax_key)

CFG = LlamaConfig(n_layers=2, hidden=64, n_heads=4, head_dim=16, inter=64, vocab=64, cluster=2)
PREFILL, STEPS = 9, 3


class OracleOps:
    """tp_step ops on one rank: numpy oracle compute on the rank's shard, gloo collectives."""

    def __init__(self, cfg, shard, rank, world, cs):
        self.cfg, self.sh, self.rank, self.world, self.cs = cfg, shard, rank, world, cs
        self.caches = [(lp_["k_cache"].copy(), lp_["v_cache"].copy()) for lp_ in shard["layers"]]
        self.cap = PREFILL + STEPS + 1
        self.caches = [(np.concatenate([k, np.zeros((k.shape[0], self.cap - k.shape[1], k.shape[2]),
                                                    np.float32)], 1),
                        np.concatenate([v, np.zeros((v.shape[0], self.cap - v.shape[1], v.shape[2]),
                                                    np.float32)], 1)) for k, v in self.caches]

    def embed(self):
        self.resid = self.sh["embed"][self.tok][None, :].astype(np.float32)

    def attn(self, l):
        L = self.sh["layers"][l]
        h = lp.rmsnorm_f16(self.resid, L["attn_norm"], self.cfg.eps)
        kc, vc = self.caches[l]
        part = lp.attention_module(h, L["w_qkv"], L["w_out"], kc, vc, self.pos, self.cfg.cluster, self.cs)
        self.acc = torch.from_numpy(np.rint(part.astype(np.float64) * 2.0 ** 32).astype(np.int64))

    def allreduce_heads(self):
        dist.all_reduce(self.acc, op=dist.ReduceOp.SUM)

    def ffn(self, l):
        L = self.sh["layers"][l]
        r = (self.resid + (self.acc.numpy().astype(np.float64) * 2.0 ** -32).astype(np.float32))
        part = lp.ffn_block(r, L["ffn_norm"], L["w1"], L["w2"], L["w3"], self.cfg.eps)
        self.resid_t = torch.from_numpy(((r if self.rank == 0 else 0.0) + part).astype(np.float32))

    def allreduce_resid(self):
        dist.all_reduce(self.resid_t, op=dist.ReduceOp.SUM)
        self.resid = self.resid_t.numpy()

    def head(self):
        hf = lp.rmsnorm_f16(self.resid, self.sh["final_norm"], self.cfg.eps)
        logits = (hf @ self.sh["lm_head"].T)[0]
        i = int(np.argmax(logits))
        V = self.sh["lm_head"].shape[0]
        self.key = torch.tensor([pack_argmax_key(logits[i], i + self.rank * V)], dtype=torch.int64)

    def allreduce_argmax(self):
        dist.all_reduce(self.key, op=dist.ReduceOp.MAX)

    def token(self):
        self.tok = unpack_argmax_key(int(self.key.item()))
        self.pos += 1


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = random_llama_params(CFG, seed=4, prefill=PREFILL)
        cs = rope_table(PREFILL + STEPS + 1, CFG.head_dim, CFG.rope_theta)
        ops = OracleOps(CFG, shard_params(params, rank, world), rank, world, cs)
        ops.tok, ops.pos = 5, PREFILL
        toks, resids = [], []
        for _ in range(STEPS):
            tp_step(ops, CFG.n_layers)
            toks.append(ops.tok)
            resids.append(ops.resid.copy())
        q.put((rank, toks, resids))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp2_schedule_matches_single_rank_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, toks, resids = q.get(timeout=240)
        res[r] = (toks, resids)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: the single-process oracle decode loop
    params = random_llama_params(CFG, seed=4, prefill=PREFILL)
    cfg1 = CFG
    caches = []
    for L in params["layers"]:
        k = np.zeros((CFG.n_heads, PREFILL + STEPS + 1, CFG.head_dim), np.float32)
        v = np.zeros_like(k)
        k[:, :PREFILL], v[:, :PREFILL] = L["k_cache"], L["v_cache"]
        caches.append((k, v))
    params = dict(params, rope_cs=rope_table(PREFILL + STEPS + 1, CFG.head_dim, CFG.rope_theta))
    tok, pos, ref = 5, PREFILL, []
    for _ in range(STEPS):
        _, tok = lp.decode_step(params, caches, tok, pos, cfg1)
        ref.append(tok)
        pos += 1
    assert res[0][0] == res[1][0] == ref
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)  # every rank holds the identical residual stream


def test_argmax_key_order():
    vals = [-3.5, -0.0, 0.0, 1e-30, 2.0, 2.0, -np.inf]
    keys = [pack_argmax_key(v, i) for i, v in enumerate(vals)]
    best = max(range(len(vals)), key=lambda i: keys[i])
    assert best == 4 and unpack_argmax_key(keys[best]) == 4   # max value, smallest index
    assert keys[0] < keys[1] < keys[3] < keys[4] and keys[6] < keys[0]


def test_local_config_and_domain():
    from paper_2508_18850_b200.llama import LLAMA2_7B
    for w, cl in ((1, 4), (2, 8), (4, 16), (8, 16)):
        lc = local_config(LLAMA2_7B, w)
        assert lc.n_heads == 32 // w and lc.inter == 11008 // w and lc.vocab == 32000 // w
        assert lc.cluster == cl
    with pytest.raises(Exception):
        check_tp(LLAMA2_7B, 3)
