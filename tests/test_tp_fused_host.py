"""The fused tensor-parallel protocol of csrc/decode_step.cu, restated on CPU
and run on two gloo ranks (world size 2) with the numpy oracle as compute.

Per rank the mirror keeps what the kernel keeps: residual buffers H[2], the
exchange block's three attention / FFN sum sets XA[3], XF[3] (int64, 2^-32
fixed point) and the argmax key.  A "push into every rank's block" is a
gloo SUM of the contributions ADDED into the receiving set (the kernel's
red.add), so a set that is not zeroed at the point the kernel zeroes it
carries stale sums into a later layer and the result breaks.  The schedule:

    step start : H[0] = embed; zero XA[0], XF[0]; key = 0;     cross barrier
    layer l    : h_l = H[(l-1)&1] + XA[(l-1)%3] + XF[(l-1)%3]  (l > 0; H[0] at l = 0)
                 H[l&1] = h_l; zero XA[(l+1)%3], XF[(l+1)%3]
                 attention(h_l) -> fixed point -> XA[l%3] += sum over ranks; cross barrier
                 ffn(H[l&1] + XA[l%3]) partial -> fixed point -> XF[l%3] += sum;  cross barrier
    head       : h_L -> local logits -> key = MAX over ranks (packed (logit, -index))

Must reproduce the single-process oracle decode (tokens equal, residuals
equal across ranks)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import llama_port as lp
from paper_2508_18850_b200.llama import LlamaConfig, random_llama_params, rope_table
from paper_2508_18850_b200.tp import pack_argmax_key, shard_params, unpack_argmax_key

CFG = LlamaConfig(n_layers=4, hidden=64, n_heads=4, head_dim=16, inter=64, vocab=64, cluster=2)
PREFILL, STEPS = 9, 4
SCALE = 2.0 ** 32


def fx(v):
    return torch.from_numpy(np.rint(np.asarray(v, np.float64) * SCALE).astype(np.int64).reshape(-1))


def unfx(t):
    return (t.numpy().astype(np.float64) / SCALE).astype(np.float32)[None, :]


class FusedMirror:
    def __init__(self, shard, rank, cs):
        self.sh, self.rank, self.cs = shard, rank, cs
        D = CFG.hidden
        self.H = [np.zeros((1, D), np.float32), np.zeros((1, D), np.float32)]
        # sets start with garbage: only the protocol's zeroing may make them usable
        self.XA = [torch.full((D,), 12345, dtype=torch.int64) for _ in range(3)]
        self.XF = [torch.full((D,), -777, dtype=torch.int64) for _ in range(3)]
        cap = PREFILL + STEPS + 1
        self.caches = []
        for L in shard["layers"]:
            k = np.zeros((L["k_cache"].shape[0], cap, CFG.head_dim), np.float32)
            v = np.zeros_like(k)
            k[:, :PREFILL], v[:, :PREFILL] = L["k_cache"], L["v_cache"]
            self.caches.append((k, v))

    def push(self, target, contrib):  # red.add of every rank's contribution into this rank's set
        t = contrib.clone()
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        target += t

    def h(self, l):
        if l == 0:
            return self.H[0]
        return (self.H[(l - 1) & 1] + unfx(self.XA[(l - 1) % 3])) + unfx(self.XF[(l - 1) % 3])

    def step(self, tok, pos):
        self.H[0] = self.sh["embed"][tok][None, :].astype(np.float32)
        self.XA[0].zero_()
        self.XF[0].zero_()
        key = torch.zeros(1, dtype=torch.int64)
        dist.barrier()
        for l, L in enumerate(self.sh["layers"]):
            hl = self.h(l)
            self.H[l & 1] = hl
            self.XA[(l + 1) % 3].zero_()
            self.XF[(l + 1) % 3].zero_()
            hn = lp.rmsnorm_f16(hl, L["attn_norm"], CFG.eps)
            kc, vc = self.caches[l]
            part = lp.attention_module(hn, L["w_qkv"], L["w_out"], kc, vc, pos, CFG.cluster, self.cs)
            self.push(self.XA[l % 3], fx(part))
            x = self.H[l & 1] + unfx(self.XA[l % 3])
            f = lp.ffn_block(x, L["ffn_norm"], L["w1"], L["w2"], L["w3"], CFG.eps)
            self.push(self.XF[l % 3], fx(f))
        hL = self.h(CFG.n_layers)
        logits = (lp.rmsnorm_f16(hL, self.sh["final_norm"], CFG.eps) @ self.sh["lm_head"].T)[0]
        i = int(np.argmax(logits))
        V = self.sh["lm_head"].shape[0]
        key += pack_argmax_key(logits[i], i + self.rank * V)
        dist.all_reduce(key, op=dist.ReduceOp.MAX)
        return unpack_argmax_key(int(key.item())), hL


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = random_llama_params(CFG, seed=6, prefill=PREFILL)
        cs = rope_table(PREFILL + STEPS + 1, CFG.head_dim, CFG.rope_theta)
        m = FusedMirror(shard_params(params, rank, world), rank, cs)
        tok, pos, toks, hs = 5, PREFILL, [], []
        for _ in range(STEPS):
            tok, hL = m.step(tok, pos)
            toks.append(tok)
            hs.append(hL)
            pos += 1
        q.put((rank, toks, hs))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_fused_tp_protocol_gloo_world2_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, toks, hs = q.get(timeout=240)
        res[r] = (toks, hs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    params = random_llama_params(CFG, seed=6, prefill=PREFILL)
    caches = []
    for L in params["layers"]:
        k = np.zeros((CFG.n_heads, PREFILL + STEPS + 1, CFG.head_dim), np.float32)
        v = np.zeros_like(k)
        k[:, :PREFILL], v[:, :PREFILL] = L["k_cache"], L["v_cache"]
        caches.append((k, v))
    params = dict(params, rope_cs=rope_table(PREFILL + STEPS + 1, CFG.head_dim, CFG.rope_theta))
    tok, pos, ref = 5, PREFILL, []
    for _ in range(STEPS):
        _, tok = lp.decode_step(params, caches, tok, pos, CFG)
        ref.append(tok)
        pos += 1
    assert res[0][0] == res[1][0] == ref
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)  # identical residual stream on every rank
