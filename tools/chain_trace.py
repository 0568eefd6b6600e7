"""Timeline of an alternating attention-module / FFN PDL chain (the engine's
launch pattern) from the kernels' %globaltimer stamps: per launch, the first
and last CTA to pass griddepcontrol.wait, and the first / last CTA to finish.

    python tools/chain_trace.py [--ctx 1024] [--layers 8]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_18850_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--layers", type=int, default=8)
a = ap.parse_args()
dev = torch.device("cuda")
D, F, nh, H, N = 4096, 11008, 32, 128, 4
L = _native.lib()
st = torch.cuda.Stream()
sp = st.cuda_stream


def rnd(*shape, s=0.02):
    return (torch.randn(*shape, device=dev) * s).half()


layers = [dict(g=rnd(D, s=1.0), w_gu=rnd(F, 2, D), w_dn=rnd(D, F), w_qkv=rnd(nh, N, 3, H // N, D),
               w_out=rnd(nh, N, D // N, H), kc=rnd(nh, a.ctx + 8, H, s=1.0), vc=rnd(nh, a.ctx + 8, H, s=1.0))
          for _ in range(a.layers)]
resid = torch.randn(1, D, device=dev)
act = torch.empty(F, device=dev, dtype=torch.float16)
bar = torch.zeros(1, device=dev, dtype=torch.int64)
accum = torch.zeros(1, D, device=dev, dtype=torch.int64)
trm = [torch.zeros(256 * 16, device=dev, dtype=torch.int64) for _ in layers]
trf = [torch.zeros(256 * 8, device=dev, dtype=torch.int64) for _ in layers]
torch.cuda.synchronize()


def launch(l, trace):
    x = layers[l]
    m = _native.MhaArgs(dtype=2, batch=1, hidden=D, n_heads=nh, head_dim=H, head_pad=H, cluster=N,
                        seq_len=a.ctx, cache_cap=a.ctx + 8,
                        flags=_native.APPEND | _native.NORM | _native.ONESHOT | _native.PDL,
                        resid=resid.data_ptr(), norm_w=x["g"].data_ptr(), eps=1e-5,
                        w_qkv=x["w_qkv"].data_ptr(), w_out=x["w_out"].data_ptr(),
                        k_cache=x["kc"].data_ptr(), v_cache=x["vc"].data_ptr(), out=None,
                        accum=accum.data_ptr(), trace=trm[l].data_ptr() if trace else None)
    _native.check(L.cfb_mha_decode(m, sp))
    f = _native.FfnArgs(dtype=2, batch=1, hidden=D, inter=F, flags=_native.NORM | _native.RESID | _native.PDL,
                        accum=accum.data_ptr(), grid=0, eps=1e-5, resid=resid.data_ptr(),
                        norm_w=x["g"].data_ptr(), w_gu=x["w_gu"].data_ptr(), w_dn=x["w_dn"].data_ptr(),
                        act=act.data_ptr(), out=resid.data_ptr(), barrier=bar.data_ptr(),
                        trace=trf[l].data_ptr() if trace else None)
    _native.check(L.cfb_ffn_decode(f, sp))


for l in range(a.layers):
    launch(l, False)
torch.cuda.synchronize()
for l in range(a.layers):
    launch(l, True)
torch.cuda.synchronize()
t0 = None
rows = []
for l in range(a.layers):
    m = trm[l].view(256, 16).cpu().numpy()[:nh * N].astype(np.float64)
    f = trf[l].view(256, 8).cpu().numpy()[:148].astype(np.float64)
    if t0 is None:
        t0 = m[:, 0].min()
    rows.append({"layer": l,
                 "mha_wait_first": round((m[:, 0].min() - t0) / 1e3, 2), "mha_wait_last": round((m[:, 0].max() - t0) / 1e3, 2),
                 "mha_end_first": round((m[:, 7].min() - t0) / 1e3, 2), "mha_end_last": round((m[:, 7].max() - t0) / 1e3, 2),
                 "ffn_wait_first": round((f[:, 0].min() - t0) / 1e3, 2), "ffn_wait_last": round((f[:, 0].max() - t0) / 1e3, 2),
                 "ffn_norm_done_med": round((np.median(f[:, 1]) - t0) / 1e3, 2),
                 "ffn_gu_done_min": round((f[:, 2].min() - t0) / 1e3, 2),
                 "ffn_gu_done_med": round((np.median(f[:, 2]) - t0) / 1e3, 2),
                 "ffn_gu_done_max": round((f[:, 2].max() - t0) / 1e3, 2),
                 "ffn_barrier_median": round((np.median(f[:, 3]) - t0) / 1e3, 2),
                 "ffn_actload_med": round((np.median(f[:, 4]) - t0) / 1e3, 2),
                 "ffn_end_first": round((f[:, 5].min() - t0) / 1e3, 2), "ffn_end_last": round((f[:, 5].max() - t0) / 1e3, 2)})
for r in rows:
    print(json.dumps(r))
print(json.dumps({"per_layer_us": round((rows[-1]["ffn_end_last"] - rows[1]["ffn_end_last"]) / (a.layers - 2), 2)}))
