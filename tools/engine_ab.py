"""A/B of the two B=1 engines (layered vs persistent) on Llama2-7B random
weights: CUDA-graph TPOT per context, plus (optionally) the persistent
engine's per-phase trace.  python tools/engine_ab.py [--ctx 1024,16384] [--trace]"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,16384")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--engines", default="layered,persistent,persistent_flat")
ap.add_argument("--trace", action="store_true")
args = ap.parse_args()
ctxs = [int(c) for c in args.ctx.split(",")]
cap = max(ctxs) + 64
res = {}
for eng in args.engines.split(","):
    # "persistent_paged" / "persistent_pagedpm": the persistent engine on a shuffled
    # 128-position page pool, head-major / page-major
    paged = "_paged" in eng
    cfg = dataclasses.replace(LLAMA2_7B, engine=eng.split("_paged")[0])
    m = LlamaDecoder.random(cfg, cache_cap=cap, seed=1)
    if paged:
        # "..._pagedseq": pages in logical order (an allocator's best case)
        m.page_kv(seed=1, layout="page_major" if eng.endswith("pm") else "head_major",
                  shuffle=not eng.endswith("seq"))
        torch.cuda.empty_cache()
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
        st = m.stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            m.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.steps
        b = cfg.step_bytes(ctx + args.steps // 2)
        res[f"{eng}@{ctx}"] = {"tpot_us": round(us, 1), "tb_s": round(b / us / 1e6, 3)}
        print(eng, ctx, res[f"{eng}@{ctx}"], flush=True)
        if args.trace and cfg.engine != "layered":
            tr = m.set_trace(True)
            m.set_state(ctx, 1)
            m.step()
            torch.cuda.synchronize()
            t = tr.cpu().numpy().astype(np.float64)  # [L][G][8]
            t0 = t[0, :, 0].min()
            # per layer: phase durations (median over CTAs) and spread of layer end
            names = ["qkv", "attn", "oproj", "bar1", "gateup", "down", "bar2"]
            d = np.diff(t, axis=2)  # [L][G][7]
            med = np.median(d, axis=1).mean(axis=0) / 1e3
            spread = (t[:, :, 6].max(axis=1) - t[:, :, 6].min(axis=1)).mean() / 1e3
            layer = np.diff(np.median(t[:, :, 0], axis=1)).mean() / 1e3
            res[f"trace_{eng}@{ctx}"] = {"phase_us_median": dict(zip(names, np.round(med, 2).tolist())),
                                   "layer_us": round(float(layer), 2),
                                   "down_end_spread_us": round(float(spread), 2)}
            print(json.dumps(res[f"trace_{eng}@{ctx}"]), flush=True)
            m.set_trace(False)
            m.capture()
    del m
    torch.cuda.empty_cache()
print(json.dumps(res))
