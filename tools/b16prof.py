"""One batch-16 Llama2-7B greedy step (ctx from argv, default 1024) for ncu
launch lists: warm-up, then a single eager decode_step between markers."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200.batched import BatchedLlama  # noqa: E402
from paper_2508_18850_b200.llama import LLAMA2_7B  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = BatchedLlama.random(LLAMA2_7B, cache_cap=ctx + 16, seed=0)
m.random_head(LLAMA2_7B.vocab)
m.set_positions([ctx] * 16)
m.decode_step()
torch.cuda.synchronize()
m.decode_step()
torch.cuda.synchronize()
