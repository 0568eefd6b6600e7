"""Per-rank shard of the tensor-parallel Llama decode on ONE B200: TPOT and the
per-phase trace of the persistent step kernel for each engine, so the TP >= 4
under-fill (few heads per rank) is visible phase by phase.
    python tools/tp_shard_trace.py [--tp 1,2,4,8] [--ctx 1024,16384]
                                   [--engines persistent,persistent_flat]"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import trace_phases  # noqa: E402
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402
from paper_2508_18850_b200.tp_fused import fused_local_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,16384")
ap.add_argument("--tp", default="1,2,4,8")
ap.add_argument("--engines", default="persistent,persistent_flat")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--clusters", default="", help="per-TP cluster override, e.g. 1:4,2:4,4:8,8:16")
a = ap.parse_args()
ctxs = [int(c) for c in a.ctx.split(",")]
cap = max(ctxs) + 64
res = []


def busy_phases(m, ctx):
    """Per-phase us over the CTAs that run attention work (qkv phase > 0.5 us):
    median and max, mean over layers."""
    import numpy as np
    tr = m.set_trace(True)
    m.set_state(ctx, 1)
    m.step()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.float64)
    m.set_trace(False)
    d = np.diff(t, axis=2) / 1e3  # [L][G][7]
    busy = d[:, :, 0].mean(axis=0) > 0.5
    names = ["qkv_gemv", "attention", "o_proj", "barrier_attn", "gate_up", "barrier_ffn", "down_and_barrier"]
    db = d[:, busy, :]
    return {"n": int(busy.sum()),
            "median": {n: round(float(v), 2) for n, v in zip(names, np.median(db, axis=1).mean(axis=0))},
            "max": {n: round(float(v), 2) for n, v in zip(names, db.max(axis=1).mean(axis=0))}}


for eng in a.engines.split(","):
    for T in [int(t) for t in a.tp.split(",")]:
        cfg = dataclasses.replace(LLAMA2_7B, n_layers=a.layers, engine=eng)
        lcfg = fused_local_config(cfg, T) if T > 1 else cfg
        ov = dict(kv.split(":") for kv in a.clusters.split(",") if kv)
        if str(T) in ov:
            lcfg = dataclasses.replace(lcfg, cluster=int(ov[str(T)]))
        m = LlamaDecoder.random(lcfg, cap, seed=1, embed_vocab=cfg.vocab)
        m.set_state(ctxs[0], 1)
        m.step()
        torch.cuda.synchronize()
        m.set_state(ctxs[0], 1)
        m.capture()
        for ctx in ctxs:
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
            us = e0.elapsed_time(e1) * 1e3 / a.steps
            bytes_ = lcfg.step_bytes(ctx)
            r = {"engine": eng, "tp": T, "ctx": ctx, "tpot_us": round(us, 1),
                 "cluster": lcfg.cluster, "gbs": round(bytes_ / us / 1e3, 1),
                 "trace": trace_phases(m, ctx), "busy_ctas": busy_phases(m, ctx)}
            res.append(r)
            print(json.dumps(r), flush=True)
        del m
        torch.cuda.empty_cache()
print(json.dumps(res))
