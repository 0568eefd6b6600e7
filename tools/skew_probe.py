"""Per-CTA skew of the persistent engine (trace stamps): which CTAs finish each
phase last, and is it the same CTAs every layer?"""
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402

eng = sys.argv[1] if len(sys.argv) > 1 else "persistent"
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = dataclasses.replace(LLAMA2_7B, engine=eng)
m = LlamaDecoder.random(cfg, cache_cap=ctx + 64, seed=1)
tr = m.set_trace(True)
out = {}
for rep in range(3):
    m.set_state(ctx, 1)
    m.step()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.float64)  # [L][G][8]
    rel = t - t[:, :, :1].min(axis=1, keepdims=True)  # vs the layer's first start
    G = t.shape[1]
    # phase k end (stamp k) per CTA relative to the layer start, us
    ends = {name: rel[:, :, k] / 1e3 for name, k in
            (("qkv_end", 1), ("attn_end", 2), ("oproj_end", 3), ("gateup_end", 5), ("down_start", 6))}
    dur_gu = (t[:, :, 5] - t[:, :, 4]) / 1e3
    dur_dn = (t[:, :, 7] - t[:, :, 6]) / 1e3
    dur_at = (t[:, :, 3] - t[:, :, 0]) / 1e3
    rank_gu = np.argsort(dur_gu.mean(axis=0))
    out[f"rep{rep}"] = {
        "spread_us": {k: round(float((v.max(axis=1) - v.min(axis=1)).mean()), 2) for k, v in ends.items()},
        "p50_p100_us": {k: [round(float(np.median(v, axis=1).mean()), 2), round(float(v.max(axis=1).mean()), 2)]
                        for k, v in ends.items()},
        "gateup_dur_fastest5": [(int(c), round(float(dur_gu.mean(axis=0)[c]), 2)) for c in rank_gu[:5]],
        "gateup_dur_slowest5": [(int(c), round(float(dur_gu.mean(axis=0)[c]), 2)) for c in rank_gu[-5:]],
        "slowest_gateup_cta_per_layer": [int(x) for x in dur_gu.argmax(axis=1)[:12]],
        "attn_dur_slowest5": [(int(c), round(float(dur_at.mean(axis=0)[c]), 2))
                              for c in np.argsort(dur_at.mean(axis=0))[-5:]],
        "corr_gateup_layers": round(float(np.corrcoef(dur_gu[1:-1:2].mean(axis=0), dur_gu[2::2].mean(axis=0))[0, 1]), 3),
        "down_dur_mean": round(float(dur_dn.mean()), 2),
    }
    print(json.dumps(out[f"rep{rep}"]), flush=True)
