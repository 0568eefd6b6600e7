"""Kernel-level timing of the fused MoE launch at DeepSeek-V2-Lite dims.

    python tools/moebench.py [--layers 4] [--reps 64] [--batch 1]
Avg µs per launch and GB/s of algorithmic bytes (router + top-k routed +
shared experts), CUDA events on the launching stream, cycling through
`layers` independent weight sets and token rows so no launch reuses L2 data.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200.moe import MoeWorkspace, moe_launch, random_moe_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--reps", type=int, default=64)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--pdl", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda")
D, E, K, F, NS = 2048, 64, 6, 1408, 2
ws_ = [random_moe_device(D, E, F, NS, K, seed=s) for s in range(a.layers)]
B = a.batch
ws = MoeWorkspace(ws_[0], B)
resid = [torch.randn(B, D, device=dev) for _ in range(a.layers)]
g = torch.ones(D, device=dev, dtype=torch.float16)
out = torch.empty(B, D, device=dev)
st = torch.cuda.Stream()
torch.cuda.synchronize()


def run(i):
    moe_launch(ws_[i % a.layers], ws, out, resid=resid[i % a.layers], norm_w=g, pdl=a.pdl,
               grid=a.grid, stream=st)


with torch.cuda.stream(st):
    for i in range(8):
        run(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(a.reps):
        run(i)
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / a.reps
idx = ws.route_idx.cpu().tolist()
# algorithmic bytes: router + union of routed experts + shared
U = len({e for row in idx for e in row})
nbytes = 2 * (E * D + 3 * D * (U * F + NS * F))
tr = torch.zeros(148, 16, device=dev, dtype=torch.int64)
with torch.cuda.stream(st):
    moe_launch(ws_[0], ws, out, resid=resid[0], norm_w=g, grid=a.grid, stream=st, trace=tr)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype("float64")
t = t[t[:, 0] > 0]
import numpy as np  # noqa: E402
rel = np.where(t[:, :14] > 0, (t[:, :14] - t[:, :1]) / 1e3, np.nan)  # globaltimer ns -> us
names = ["start", "norm", "router", "routed", "shared_gu", "shared_dn", "routed_gu", "routed_dn",
         "atomics", "last_cta", "end", "r_polled", "r_loaded", "r_ranked"]
print("cta0", [round(float(x), 2) for x in rel[0]], "cta77", [round(float(x), 2) for x in rel[77]])
print(json.dumps({"trace_us_mean": {n: round(float(np.nanmean(rel[:, k])), 2) for k, n in enumerate(names)},
                  "trace_us_max": {n: round(float(np.nanmax(rel[:, k])), 2) for k, n in enumerate(names)}}))
print(json.dumps({"kernel": "moe_kernel", "batch": B, "us": round(us, 2),
                  "GBps": round(nbytes / us / 1e3, 1), "bytes": nbytes, "experts_streamed": U}))
