"""Standalone final RMSNorm + LM head + argmax launches (for ncu).

The B=1 Llama engine runs its LM head inside the step kernel; the layered
`lm_head_kernel` (`cfb_lm_head_argmax`) is the DeepSeek model's (V = 102,400,
D = 2048) and the layered Llama engine's (V = 32,000, D = 4096).  Runs 3
launches of each shape, weights device-drawn:
    ncu --set full -k regex:lm_head -s 1 -c 1 python tools/profile_lm_head.py
Prints the algorithmic bytes (V x D fp16 weights + the D-vector reads + V fp32
logits written) and the CUDA-event time of the warm launches."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200 import _native  # noqa: E402
from paper_2508_18850_b200.layouts import row_tiles  # noqa: E402

SHAPES = [("llama2-7b", 32000, 4096), ("deepseek-v2-lite", 102400, 2048)]
only = sys.argv[1] if len(sys.argv) > 1 else None
dev = _native.require_cuda()
L = _native.lib()
out = []
for name, V, D in SHAPES:
    if only and only != name:
        continue
    g = torch.Generator(device=dev).manual_seed(1)
    w = row_tiles((torch.randn(V, D, device=dev, generator=g) * D ** -0.5).half())
    r = torch.randn(1, D, device=dev, generator=g)
    gw = torch.ones(D, device=dev, dtype=torch.float16)
    logits = torch.empty(1, V, device=dev, dtype=torch.float32)
    cv = torch.empty(1024, device=dev, dtype=torch.float32)
    ci = torch.empty(1024, device=dev, dtype=torch.int32)
    ticket = torch.zeros(1, device=dev, dtype=torch.int32)
    tok = torch.empty(1, device=dev, dtype=torch.int32)
    a = _native.LmArgs(dtype=2, batch=1, hidden=D, vocab=V, grid=0, eps=1e-5,
                       resid=r.data_ptr(), norm_w=gw.data_ptr(), w=w.data_ptr(),
                       logits=logits.data_ptr(), cand_val=cv.data_ptr(), cand_idx=ci.data_ptr(),
                       ticket=ticket.data_ptr(), token_out=tok.data_ptr(), step_pos=None)
    sp = _native.stream_ptr()
    flush = torch.empty(256 << 20, device=dev, dtype=torch.uint8)
    ts = []
    for i in range(3):
        flush.zero_()  # weights cold in L2 (larger-than-L2 write)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(L.cfb_lm_head_argmax(ctypes.byref(a), sp))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ref = int(torch.argmax(logits[0]).item())  # the kernel's token is the first-index argmax of its logits
    assert int(tok[0]) == ref, (int(tok[0]), ref)
    nbytes = V * D * 2 + D * 4 + D * 2 + V * 4
    us = min(ts[1:])
    out.append({"model": name, "vocab": V, "hidden": D, "bytes": nbytes, "us_warm_best": round(us, 2),
                "gbs": round(nbytes / us / 1e3, 1)})
print(json.dumps(out))
