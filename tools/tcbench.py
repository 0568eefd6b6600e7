"""tcgen05 batch-16 projection timing at Llama2-7B FFN shapes (CUDA events,
cycling weight sets so nothing is L2-resident)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200.tc import TcProjection  # noqa: E402

res = []
for M, K in ((22016, 4096), (4096, 11008), (12288, 4096), (4096, 4096)):
    ps = [TcProjection(torch.randn(M, K, device="cuda") * K ** -0.5) for _ in range(3)]
    x = torch.randn(16, K, device="cuda").half()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for p in ps:
            p.launch(x, pdl=True, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 30
        e0.record(st)
        for r in range(reps):
            ps[r % 3].launch(x, pdl=True, stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    nbytes = M * K * 2
    res.append({"M": M, "K": K, "us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1),
                "TFLOPs": round(2 * 16 * M * K / us / 1e6, 1)})
    del ps
    torch.cuda.empty_cache()
from paper_2508_18850_b200.tc import TcFfnB16  # noqa: E402

D, F = 4096, 11008
ffns = [TcFfnB16(torch.randn(F, D, device="cuda") * D ** -0.5, torch.randn(F, D, device="cuda") * D ** -0.5,
                 torch.randn(D, F, device="cuda") * F ** -0.5, torch.ones(D, device="cuda")) for _ in range(3)]
resid = torch.randn(16, D, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for f in ffns:
        f.launch(resid, pdl=True, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for r in range(30):
        ffns[r % 3].launch(resid, pdl=True, stream=st)
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 30
print(json.dumps({"tc_gemm_b16": res, "ffn_b16": {"us": round(us, 2), "GBps": round(ffns[0].weight_bytes / us / 1e3, 1),
                                                  "tokens_per_s": round(16 / us * 1e6, 1)}}))
