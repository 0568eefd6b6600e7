"""A/B of the persistent step kernel's ring depth (8 KB slots per consumer
warp: 3 = 192 KB, 2 = 128 KB per CTA), alternating, CUDA-graph TPOT.
    python tools/ring_ab.py [--ctx 1024,4096,16384] [--spw 3,2] [--reps 2]"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,4096,16384")
ap.add_argument("--spw", default="3,2")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--engine", default="persistent")
ap.add_argument("--pool", default="", help="A/B pool tiles per CTA instead of ring depth, e.g. 4,8,2")
a = ap.parse_args()
ctxs = [int(c) for c in a.ctx.split(",")]
cfg = dataclasses.replace(LLAMA2_7B, engine=a.engine)
m = LlamaDecoder.random(cfg, max(ctxs) + 64, seed=1)
res = {}
for rep in range(a.reps):
    for spw in [int(s) for s in (a.pool or a.spw).split(",")]:
        if a.pool:
            m.set_pool_tiles(spw)
        else:
            m.set_ring_slots(spw)
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
            res.setdefault(f"spw{spw}@{ctx}", []).append(round(us, 1))
            print("spw", spw, "ctx", ctx, round(us, 1), flush=True)
print(json.dumps(res))
