"""One eager persistent decode step of Llama2-7B at a given context (for ncu).
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:llama_step --launch-skip 1 -c 1 python tools/profile_step_kernel.py 1024 [engine] [paged]"""
import dataclasses
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eng = sys.argv[2] if len(sys.argv) > 2 else "persistent"
m = LlamaDecoder.random(dataclasses.replace(LLAMA2_7B, engine=eng), cache_cap=ctx + 8, seed=1)
if len(sys.argv) > 3 and sys.argv[3] == "paged":  # shuffled head-major page pool
    m.page_kv(seed=1)
m.set_plain_launch(True)  # ncu cannot replay cooperative cluster launches
for _ in range(2):
    m.set_state(ctx, 1)
    m.step()
torch.cuda.synchronize()
print("bytes", LLAMA2_7B.step_bytes(ctx))
