"""Sweep CFB_OPT_L2_PREFETCH (bytes per CTA prefetched into L2 past the smem
ring at each grid barrier) on the Llama2-7B persistent engine.
    python tools/prefetch_ab.py [--ctx 1024,16384] [--pf 0,131072,262144] [--engine persistent]"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,16384")
ap.add_argument("--pf", default="0,65536,131072,262144,393216,524288")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--engine", default="persistent")
a = ap.parse_args()
ctxs = [int(c) for c in a.ctx.split(",")]
cfg = dataclasses.replace(LLAMA2_7B, engine=a.engine)
m = LlamaDecoder.random(cfg, cache_cap=max(ctxs) + 64, seed=1)
m.set_state(ctxs[0], 1)
m.step()
torch.cuda.synchronize()
res = {}
for rnd in range(a.rounds):  # interleaved rounds: box drift shows up as round-to-round spread
    for pf in [int(x) for x in a.pf.split(",")]:
        m.set_l2_prefetch(pf)
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
            res.setdefault(f"{pf}@{ctx}", []).append(round(us, 1))
            print(rnd, pf, ctx, round(us, 1), flush=True)
print(json.dumps({k: {"tpot_us": v, "best": min(v)} for k, v in res.items()}))
