"""Per-rank shard compute of the tensor-parallel DeepSeek block and Llama
layer on ONE GPU (no all-reduce: the reductions are no-ops).  A lower bound
for one rank's time at TP 2/4/8, not a multi-GPU measurement (that is the
driver's torchrun scaling run of bench.py)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200.deepseek import LITE  # noqa: E402
from paper_2508_18850_b200.tp import TPDeepSeekBlock, deepseek_local_dims  # noqa: E402

res = []
for world in [int(w) for w in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]:
    for ctx in [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1024,16384").split(",")]:
        nop = (lambda t: None)
        blocks = [TPDeepSeekBlock.random(LITE, 0, world, ctx, seed=l, reduce_int=nop, reduce_f32=nop)
                  for l in range(4)]
        resid = torch.full((1, LITE.hidden), 0.5, device="cuda")
        st = torch.cuda.Stream()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            for b in blocks:
                b.launch(resid)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for b in blocks:
                b.launch(resid)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(16):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 64
        ld = deepseek_local_dims(LITE, world)
        res.append({"model": "deepseek_block", "tp": world, "ctx": ctx, "rank_shard_us": round(us, 2),
                    "rank_bytes": ld.block_bytes(ctx), "rank_hbm_gbs": round(ld.block_bytes(ctx) / us / 1e3, 1)})
        print(json.dumps(res[-1]), flush=True)
        del g, blocks
        torch.cuda.empty_cache()
print(json.dumps({"tp_shard_compute": res}))
