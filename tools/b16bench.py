"""Batch-16 independent-sequence Llama2-7B decode on the tcgen05 path:
32 layers (QKV/O/FFN projections on tcgen05, split-KV attention per sequence),
CUDA-graph replay, per-step latency and tokens/s at several contexts."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200.batched import BatchedLlama  # noqa: E402
from paper_2508_18850_b200.llama import LLAMA2_7B  # noqa: E402

ctxs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1024,4096").split(",")]
steps = 10
out = []
for ctx in ctxs:
    m = BatchedLlama.random(LLAMA2_7B, cache_cap=ctx + 3 * steps + 8, seed=0)
    m.set_positions([ctx] * 16)
    m.step()
    torch.cuda.synchronize()
    m.set_positions([ctx] * 16)
    m.capture()
    for _ in range(3):
        m.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    for _ in range(steps):
        m.replay()
    e1.record(m.stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    nbytes = m.step_bytes(ctx + 3 + steps // 2)
    out.append({"ctx": ctx, "step_us": round(us, 1), "tokens_per_s": round(16e6 / us, 1),
                "hbm_gbs": round(nbytes / us / 1e3, 1), "bytes": nbytes})
    print(json.dumps(out[-1]), flush=True)
    del m
    torch.cuda.empty_cache()
print(json.dumps({"batch16_llama_stack": out}))
