"""Kernel-level timing of the fused FFN and attention modules at Llama2-7B dims.

    python tools/kbench.py [--ctx 1024] [--reps 64]
Prints avg µs per launch and GB/s (algorithmic bytes / time), CUDA events,
cycling through 32 layers' worth of weights so nothing stays in L2.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2508_18850_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--reps", type=int, default=64)
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--cluster", type=int, default=4)
ap.add_argument("--no-pdl", action="store_true")
ap.add_argument("--dbg", type=int, default=0)
ap.add_argument("--mode", default="oneshot", choices=["oneshot", "merged", "two_pass"])
a = ap.parse_args()
a.pdl = 0 if a.no_pdl else _native.PDL
a.mode = {"oneshot": _native.ONESHOT, "merged": _native.STATS_MERGED, "two_pass": 0}[a.mode]
dev = torch.device("cuda")
D, F, nh, H, N = 4096, 11008, 32, 128, a.cluster
L = _native.lib()
st = torch.cuda.Stream()
sp = st.cuda_stream


def rnd(*shape, s=0.02):
    return (torch.randn(*shape, device=dev) * s).half()


layers = [dict(g=rnd(D, s=1.0), w_gu=rnd(F, 2, D), w_dn=rnd(D, F), w_qkv=rnd(nh, N, 3, H // N, D),
               w_out=rnd(nh, N, D // N, H), kc=rnd(nh, a.ctx + 8, H, s=1.0), vc=rnd(nh, a.ctx + 8, H, s=1.0))
          for _ in range(a.layers)]
resid = torch.randn(1, D, device=dev)
out = torch.empty(1, D, device=dev)
act = torch.empty(F, device=dev, dtype=torch.float16)
bar = torch.zeros(1, device=dev, dtype=torch.int64)
accum = torch.zeros(1, D, device=dev, dtype=torch.int64)
pos = torch.tensor([a.ctx], device=dev, dtype=torch.int32)
torch.cuda.synchronize()


def ffn(l):
    return _native.FfnArgs(dtype=2, batch=1, hidden=D, inter=F,
                           flags=_native.NORM | _native.RESID | a.pdl, accum=accum.data_ptr(),
                           grid=0, eps=1e-5, resid=resid.data_ptr(), norm_w=l["g"].data_ptr(),
                           w_gu=l["w_gu"].data_ptr(), w_dn=l["w_dn"].data_ptr(), act=act.data_ptr(),
                           out=out.data_ptr(), barrier=bar.data_ptr())


def mha(l):
    return _native.MhaArgs(dtype=2, batch=1, hidden=D, n_heads=nh, head_dim=H, head_pad=H, cluster=N,
                           seq_len=a.ctx, cache_cap=a.ctx + 8,
                           flags=_native.APPEND | _native.NORM | a.mode | a.pdl | a.dbg,
                           resid=resid.data_ptr(),
                           norm_w=l["g"].data_ptr(), eps=1e-5, w_qkv=l["w_qkv"].data_ptr(),
                           w_out=l["w_out"].data_ptr(), k_cache=l["kc"].data_ptr(),
                           v_cache=l["vc"].data_ptr(), out=None, accum=accum.data_ptr())


def timeit(fn, args, nbytes):
    for x in args[:4]:
        _native.check(fn(x, sp))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(a.reps):
        _native.check(fn(args[i % len(args)], sp))
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    return {"us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1)}


res = {
    "ffn": timeit(L.cfb_ffn_decode, [ffn(l) for l in layers], 3 * D * F * 2 + 2 * D),
    "mha": timeit(L.cfb_mha_decode, [mha(l) for l in layers],
                  (D * 3 * nh * H + nh * H * D) * 2 + 2 * nh * H * 2 * a.ctx),
}
print(json.dumps(res))

# ---- per-CTA phase timeline (globaltimer stamps, ns) of one launch each
if "--trace" in sys.argv or True:
    import numpy as np
    tr = torch.zeros(256 * 8, device=dev, dtype=torch.int64)
    fa = ffn(layers[0]); fa.trace = tr.data_ptr()
    _native.check(L.cfb_ffn_decode(fa, sp)); torch.cuda.synchronize()
    t = tr.view(256, 8).cpu().numpy()[:148, :6].astype(np.float64)
    t0 = t[:, 0].min()
    names = ["start", "norm", "gateup", "barrier", "actload", "down"]
    print("ffn timeline us (min/median/max per stamp):",
          {n: (round((t[:, k].min() - t0) / 1e3, 2), round((np.median(t[:, k]) - t0) / 1e3, 2),
               round((t[:, k].max() - t0) / 1e3, 2)) for k, n in enumerate(names)})
    tr = torch.zeros(256 * 16, device=dev, dtype=torch.int64)
    ma = mha(layers[0]); ma.trace = tr.data_ptr()
    torch.cuda.synchronize()
    for i in range(1, 4):  # traced launch inside a warm PDL chain, like the engine
        _native.check(L.cfb_mha_decode(mha(layers[i]), sp))
    _native.check(L.cfb_mha_decode(ma, sp)); torch.cuda.synchronize()
    t = tr.view(256, 16).cpu().numpy()[:nh * N].astype(np.float64)
    t0 = t[:, 0].min()
    names = ["start", "norm", "qkv", "gather", "attn", "stats", "oproj", "end", "cwait", "push",
             "xchg", "attn0", "kvdone", "newtok"]
    print("mha timeline us (min/median/max per stamp):",
          {n: (round((t[:, k].min() - t0) / 1e3, 2), round((np.median(t[:, k]) - t0) / 1e3, 2),
               round((t[:, k].max() - t0) / 1e3, 2)) for k, n in enumerate(names)})
    import os
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/mha_trace_ctx{a.ctx}.npy", (t - t0) / 1e3)
    print("oproj math cycles (warp 0) median", np.median(t[:, 14]), "items", np.median(t[:, 15]))
