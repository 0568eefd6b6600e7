"""Drive a few eager Llama2-7B decode steps for ncu (no CUDA graph, no timing).

    ncu ... python tools/profile_step.py [--ctx 1024] [--steps 2] [--layers 32]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2508_18850_b200.llama import LlamaConfig, LlamaDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--cluster", type=int, default=4)
a = ap.parse_args()
cfg = LlamaConfig(n_layers=a.layers, cluster=a.cluster)
m = LlamaDecoder.random(cfg, cache_cap=a.ctx + a.steps + 4, seed=0)
m.set_state(a.ctx, 1)
for _ in range(a.steps):
    m.step()
torch.cuda.synchronize()
print("done", m.token())
