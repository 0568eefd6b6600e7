"""split_token vs split_head on the GPU (the paper's App. B.2 comparison,
PAPER.md:1229-1234): one Llama2-7B attention module (32 heads x 128, D=4096,
B=1, f16) through the drop-in API kernels at several contexts, cluster 4.
Kernel time by CUDA events around the C-ABI launch (weights already packed
on the device; the reference-API wrappers' packing is excluded)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200 import _native  # noqa: E402

L = _native.lib()
dev = torch.device("cuda")
D, nh, H, N = 4096, 32, 128, 4
out = []
for S in (1024, 4096):
    x = (torch.randn(1, D, device=dev)).half()
    # split_head: reference layouts
    wqkv = (torch.randn(nh, D, 3 * H, device=dev) * D ** -0.5).half()
    wo = (torch.randn(nh, H, D, device=dev) * H ** -0.5).half()
    kc = torch.randn(nh, S, H, device=dev).half()
    vc = torch.randn(nh, S, H, device=dev).half()
    o = torch.empty(1, D, device=dev)
    acc = torch.zeros(1, D, device=dev, dtype=torch.int64)
    sh = _native.SplitHeadArgs(dtype=2, batch=1, hidden=D, n_heads=nh, head_dim=H, cluster=N,
                               seq_len=S, flags=_native.APPEND, x=x.data_ptr(), w_qkv=wqkv.data_ptr(),
                               w_out=wo.data_ptr(), k_cache=kc.data_ptr(), v_cache=vc.data_ptr(),
                               out=o.data_ptr(), accum=acc.data_ptr(), stats=None, traffic=None)
    # split_token: kernel layouts (random, same byte counts)
    wq2 = (torch.randn(nh, N, 3 * H // N // 4, D // 8, 4, 8, device=dev) * D ** -0.5).half()
    wo2 = (torch.randn(nh, N, D // N, H, device=dev) * H ** -0.5).half()
    kc2 = torch.randn(nh, S + 8, H, device=dev).half()
    vc2 = torch.randn(nh, S + 8, H, device=dev).half()
    st = _native.MhaArgs(dtype=2, batch=1, hidden=D, n_heads=nh, head_dim=H, head_pad=H, cluster=N,
                         seq_len=S, cache_cap=S + 8, flags=_native.APPEND, x=x.data_ptr(),
                         w_qkv=wq2.data_ptr(), w_out=wo2.data_ptr(), k_cache=kc2.data_ptr(),
                         v_cache=vc2.data_ptr(), out=o.data_ptr(), accum=acc.data_ptr())
    sp = torch.cuda.current_stream().cuda_stream
    res = {"ctx": S}
    for name, fn, a in (("split_head", L.cfb_splithead_decode, sh), ("split_token", L.cfb_mha_decode, st)):
        try:
            for _ in range(3):
                _native.check(fn(a, sp))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                _native.check(fn(a, sp))
            e1.record()
            torch.cuda.synchronize()
            res[name + "_us"] = round(e0.elapsed_time(e1) * 1e3 / 20, 2)
        except Exception as exc:  # e.g. split_head's S x B score reduce exceeding smem
            res[name + "_us"] = None
            res[name + "_error"] = str(exc)[:120]
    out.append(res)
print(json.dumps({"dataflow_compare": out}))
