"""DeepSeek-V2-Lite-shaped block timing (BASELINE.json config #3).

    python tools/dsbench.py [--contexts 1024,4096,16384] [--layers 4] [--reps 32]
µs per block (fused_mla + fused MoE, PDL-chained, CUDA-graph replay of
`layers` distinct blocks so nothing is reused from L2) and achieved GB/s of
algorithmic bytes; also the two kernels alone.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200 import _native  # noqa: E402
from paper_2508_18850_b200.deepseek import LITE, DeepSeekBlock  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--contexts", default="1024,4096,16384")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--reps", type=int, default=32)
ap.add_argument("--reference-mla", action="store_true", help="reference-dataflow MLA kernel")
a = ap.parse_args()
out = []
for S in [int(c) for c in a.contexts.split(",")]:
    blocks = [DeepSeekBlock.random(LITE, S, seed=s, use_engine=not a.reference_mla)
              for s in range(a.layers)]
    st = torch.cuda.Stream()
    resid = torch.randn(1, LITE.hidden, device="cuda")
    with torch.cuda.stream(st):
        for b in blocks:
            b.launch(resid, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for b in blocks:
            b.launch(resid, stream=st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(a.reps):
            g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (a.reps * a.layers)
    nbytes = LITE.block_bytes(S)
    # kernels alone (eager, PDL chain of the same kind)
    def time_fn(fn):
        with torch.cuda.stream(st):
            for _ in range(4):
                fn()
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(a.reps):
                fn()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / a.reps
    k = [0]

    def mla_only():
        b = blocks[k[0] % a.layers]
        k[0] += 1
        b.launch_attention(resid, True, stream=st)
    mla_us = time_fn(mla_only)
    out.append({"ctx": S, "block_us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1),
                "bytes": nbytes, "mla_us": round(mla_us, 2),
                "mla_GBps": round(LITE.mla_bytes(S) / mla_us / 1e3, 1)})
    print(json.dumps(out[-1]), flush=True)
    del blocks
    torch.cuda.empty_cache()
print(json.dumps({"deepseek_block": out}))
