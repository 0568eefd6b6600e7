import sys, torch
sys.path.insert(0, '.')
from paper_2508_18850_b200.batched import BatchedLlama
from paper_2508_18850_b200.llama import LlamaConfig
cfg = LlamaConfig(n_layers=2)
m = BatchedLlama.random(cfg, cache_cap=1100, seed=0)
m.set_positions([1024] * 16)
for _ in range(3):
    m.step()
torch.cuda.synchronize()
