"""Tensor-parallel DeepSeek block schedule on CPU (gloo, world 2 and 4): each
rank runs the numpy oracle on its shard (``tp.shard_deepseek``: MLA heads,
expert intermediate rows; latent cache, W_kv and router replicated) in the
order ``tp.TPDeepSeekBlock.launch`` uses - attention partial -> SUM ->
MoE partial (residual + attention on rank 0 only) -> SUM - and must reproduce
the single-process oracle block (oracle/deepseek_port.block)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import clusterdec_port as cp
from oracle import deepseek_port as dp
from oracle.llama_port import rmsnorm_f16
from paper_2508_18850_b200.deepseek import DeepSeekDims
from paper_2508_18850_b200.exceptions import DimensionError
from paper_2508_18850_b200.tp import check_tp_deepseek, deepseek_local_dims, shard_deepseek

DIMS = DeepSeekDims(hidden=64, n_heads=4, head_dim=16, kv_rank=32, n_experts=8, top_k=2, inter=32,
                    n_shared=1, cluster=2)
S = 20
KEYS = ("w_q", "w_up", "w_kv", "w_down", "w_out", "kv_cache")


def _inputs():
    mla = cp.gen_mla(1, DIMS.hidden, DIMS.n_heads, DIMS.head_dim, S, DIMS.kv_rank, seed=3)
    moe_w = dp.gen_moe(DIMS.hidden, DIMS.n_experts, DIMS.inter, DIMS.n_shared, seed=2)
    rng = np.random.default_rng(5)
    resid = rng.standard_normal((1, DIMS.hidden)).astype(np.float32)
    g1 = dp.f16(1.0 + 0.1 * rng.standard_normal(DIMS.hidden))
    g2 = dp.f16(1.0 + 0.1 * rng.standard_normal(DIMS.hidden))
    return {k: mla[k] for k in KEYS}, moe_w, resid, g1, g2


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mla, moe_w, resid, g1, g2 = _inputs()
        _, mla_r, moe_r = shard_deepseek(DIMS, mla, moe_w, rank, world)
        h = rmsnorm_f16(resid, g1, DIMS.eps)
        attn_r = cp.fused_mla(dict(mla_r, hidden=h), DIMS.cluster, 2, "two_pass", append=True,
                              head_accum="f32")[0]
        t = torch.from_numpy(np.ascontiguousarray(attn_r, np.float32))
        dist.all_reduce(t)                                     # the int64 fixed-point SUM on the GPU
        x = resid + t.numpy()
        h2 = rmsnorm_f16(x, g2, DIMS.eps)
        y_r, idx, _, _ = dp.moe(h2, moe_r, DIMS.top_k, DIMS.routed_scale)
        out = torch.from_numpy(np.ascontiguousarray((x if rank == 0 else 0.0) + y_r, np.float32))
        dist.all_reduce(out)                                   # CFB_PARTIAL on ranks > 0
        q.put((rank, out.numpy(), np.asarray(idx)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_tp_deepseek_schedule_matches_single_rank_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, out, idx = q.get(timeout=240)
        res[r] = (out, idx)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mla, moe_w, resid, g1, g2 = _inputs()
    ref, info = dp.block(resid, mla, g1, g2, moe_w, DIMS.top_k, DIMS.cluster, DIMS.eps, DIMS.routed_scale)
    for r in range(world):
        assert np.array_equal(res[r][1], info["idx"])          # identical routing on every rank
        np.testing.assert_allclose(res[r][0], ref, rtol=1e-5, atol=1e-5)
        assert np.array_equal(res[r][0], res[0][0])             # replicated residual stream


def test_deepseek_tp_domain():
    from paper_2508_18850_b200.deepseek import LITE
    for w in (1, 2, 4, 8):
        ld = deepseek_local_dims(LITE, w)
        assert ld.n_heads * w == LITE.n_heads and ld.inter * w == LITE.inter and ld.inter % 8 == 0
    with pytest.raises(DimensionError):
        check_tp_deepseek(LITE, 3)
    with pytest.raises(DimensionError):
        check_tp_deepseek(DeepSeekDims(inter=1400), 2)   # 700 is not a multiple of 8
    mla, moe_w, _, _, _ = _inputs()
    ld, m, e = shard_deepseek(DIMS, mla, moe_w, 1, 2)
    assert m["w_q"].shape == (2, DIMS.hidden, DIMS.head_dim) and m["w_kv"].shape == mla["w_kv"].shape
    assert e["experts"][3]["gate"].shape == (16, DIMS.hidden) and e["experts"][3]["down"].shape == (DIMS.hidden, 16)
    assert np.array_equal(e["experts"][3]["up"], moe_w["experts"][3]["up"][16:32])
    assert e["shared"]["down"].shape == (DIMS.hidden, 16)
