"""Fused tensor parallel on ONE B200 (no multi-GPU box here):
  * shard : one rank's shard (nh/T heads, F/T, V/T) as a single-GPU persistent
            step on all SMs, no exchange - the per-rank compute lower bound at TP T;
  * emul  : all T ranks of the fused path on one GPU (1/T of the SMs each, the
            in-kernel all-reduces over "peer" memory on the same device):
            the same total bytes as TP1, so TPOT(emul T) - TPOT(TP1) bounds the
            protocol's cost (cross-rank barriers + fixed-point pushes).
    python tools/tp_fused_time.py [--ctx 1024,16384] [--tp 2,4,8] [--layers 32]"""
import argparse
import dataclasses
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402
from paper_2508_18850_b200.tp_fused import FusedTPLlama, emulated_grid, fused_local_config  # noqa: E402
from paper_2508_18850_b200.tp_fused import EmulatedTP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,16384")
ap.add_argument("--tp", default="2,4,8")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--engine", default="persistent")
a = ap.parse_args()
ctxs = [int(c) for c in a.ctx.split(",")]
cfg = dataclasses.replace(LLAMA2_7B, n_layers=a.layers, engine=a.engine)
cap = max(ctxs) + 64
res = {}


def time_graph(m, ctx):
    m.set_state(ctx, 1)
    for _ in range(3):
        m.replay()
    m.set_state(ctx, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    for _ in range(a.steps):
        m.replay()
    e1.record(m.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.steps


def prep(m, ctx):
    m.set_state(ctx, 1)
    m.step()
    torch.cuda.synchronize()
    m.set_state(ctx, 1)
    m.capture()


m = LlamaDecoder.random(cfg, cap, seed=1)
prep(m, ctxs[0])
for ctx in ctxs:
    res[f"tp1@{ctx}"] = round(time_graph(m, ctx), 1)
    print("tp1", ctx, res[f"tp1@{ctx}"], flush=True)
del m
torch.cuda.empty_cache()
for T in [int(t) for t in a.tp.split(",")]:
    lcfg = fused_local_config(cfg, T)
    m = LlamaDecoder.random(lcfg, cap, seed=1, embed_vocab=cfg.vocab)
    prep(m, ctxs[0])
    for ctx in ctxs:
        res[f"shard{T}@{ctx}"] = round(time_graph(m, ctx), 1)
        print("shard", T, ctx, res[f"shard{T}@{ctx}"], flush=True)
    del m
    torch.cuda.empty_cache()
    grid = emulated_grid(cfg, T)
    ranks = [FusedTPLlama(cfg, r, T, cap, seed=1, peers=True, emulated=True, grid=grid) for r in range(T)]
    ptrs = [r.xch.ptr.value for r in ranks]
    for r in ranks:
        r._attach(ptrs, emulated=True, grid=grid, timeout_s=10.0)
    tp = EmulatedTP(ranks)
    tp.set_state(ctxs[0], 1)
    tp.step()
    tp.set_state(ctxs[0], 1)
    tp.capture()
    for ctx in ctxs:
        tp.set_state(ctx, 1)
        for _ in range(3):
            tp.replay()
        tp.set_state(ctx, 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            for r in ranks:
                r.replay()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) * 1e6 / a.steps
        tp.check()
        res[f"emul{T}@{ctx}"] = round(us, 1)
        print("emul", T, ctx, res[f"emul{T}@{ctx}"], "grid/rank", grid, flush=True)
    del tp, ranks
    torch.cuda.empty_cache()
print(json.dumps(res))
