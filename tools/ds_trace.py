"""Timeline of the DeepSeek block's MLA engine (3 launches) from per-CTA
%globaltimer stamps (cfb_mla_engine_args.trace), eager PDL chain of `layers`
distinct blocks; us relative to the block's first mla_proj consumer start.
    python tools/ds_trace.py [--ctx 1024,16384] [--layers 4]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.deepseek import LITE, DeepSeekBlock  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="1024,16384")
ap.add_argument("--layers", type=int, default=4)
a = ap.parse_args()
names = {0: "proj_start", 1: "proj_norm", 2: "proj_qc", 3: "proj_barrier", 4: "proj_qlat",
         5: "attn_start", 6: "attn_q", 7: "attn_end", 8: "out_start", 14: "out_weights", 9: "out_merge",
         10: "out_barrier1", 11: "out_wdown", 12: "out_barrier2", 13: "out_end"}
moe_names = {0: "moe_start", 14: "moe_norm1", 1: "moe_norm", 2: "moe_router", 11: "moe_polled", 12: "moe_loaded",
             13: "moe_ranked", 3: "moe_routed", 7: "moe_experts", 8: "moe_atomics", 9: "moe_last",
             10: "moe_end"}
res = {}
for S in [int(c) for c in a.ctx.split(",")]:
    blocks = [DeepSeekBlock.random(LITE, S, seed=s) for s in range(a.layers)]
    for b in blocks:
        b.trace = torch.zeros(148, 16, device="cuda", dtype=torch.int64)
        b.moe_trace = torch.zeros(148, 16, device="cuda", dtype=torch.int64)
    st = torch.cuda.Stream()
    resid = torch.randn(1, LITE.hidden, device="cuda")
    for rep in range(4):
        for b in blocks:
            b.trace.zero_()
            b.moe_trace.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for b in blocks:
                b.launch(resid, stream=st)
        torch.cuda.synchronize()
    rows = []
    for b in blocks[1:]:
        t = b.trace.cpu().numpy().astype(np.float64)
        t0 = np.min(t[:, 0][t[:, 0] > 0])
        row = {}
        for k, n in names.items():
            v = t[:, k]
            v = v[v > 0]
            if len(v):
                row[n] = (float(np.median(v) - t0) / 1e3, float(np.max(v) - t0) / 1e3)
        tm = b.moe_trace.cpu().numpy().astype(np.float64)
        for k, n in moe_names.items():
            v = tm[:, k]
            v = v[v > 0]
            if len(v):
                row[n] = (float(np.median(v) - t0) / 1e3, float(np.max(v) - t0) / 1e3)
        rows.append(row)
    allnames = list(names.values()) + list(moe_names.values())
    summ = {n: [round(float(np.mean([r[n][0] for r in rows if n in r])), 2),
                round(float(np.mean([r[n][1] for r in rows if n in r])), 2)]
            for n in allnames if any(n in r for r in rows)}
    res[S] = summ
    print(S, json.dumps(summ), flush=True)
    del blocks
    torch.cuda.empty_cache()
print(json.dumps(res))
