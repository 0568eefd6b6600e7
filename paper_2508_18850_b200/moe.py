"""DeepSeek-V2 MoE layer on the GPU: one fused launch of ``csrc/moe.cu``
(router GEMV -> softmax top-k -> shared + routed SwiGLU expert GEMVs ->
weighted sum, optional RMSNorm prologue and residual epilogue).

The reference package has no MoE; the semantics are
``transformers``' ``DeepseekV2Moe`` (greedy softmax top-k, shared experts),
restated in ``oracle/deepseek_port.py`` and pinned by
``tests/golden/moe_golden.*``.  Weights are packed once into the kernel
layouts of ``include/cfb.h`` (``cfb_moe_args``) and stay resident.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .exceptions import DimensionError, ShapeMismatch
from .layouts import gate_up_tiles


def moe_segments(hidden: int) -> int:
    """Q: down-projection column segments (csrc/moe.cu moe_segments)."""
    return hidden // 512 if hidden >= 512 else 1


def down_blocks(w_down):
    """(D, F) = W_down -> [F/8][Q][8][D/Q] blocks of W_down^T (fp16)."""
    D, F = w_down.shape
    Q = moe_segments(D)
    return w_down.t().reshape(F // 8, 8, Q, D // Q).permute(0, 2, 1, 3).contiguous()


@dataclass
class MoeWeights:
    """Device-resident packed MoE weights (fp16)."""
    hidden: int
    n_experts: int
    top_k: int
    inter: int
    shared_inter: int
    routed_scale: float
    router: object       # [E][D]
    w_gu: object         # [E][F/2][D/8][4][8]
    w_dn: object         # [E][F/8][Q][8][D/Q]
    s_gu: object = None
    s_dn: object = None

    @property
    def algorithmic_bytes(self) -> int:
        """HBM bytes one B=1 launch must read: router + top_k routed experts
        + shared experts (3 matrices of D x width each), fp16."""
        D = self.hidden
        return 2 * (self.n_experts * D + 3 * D * (self.top_k * self.inter + self.shared_inter))


def pack_moe(w: dict, top_k: int, routed_scale: float = 1.0, device=None) -> MoeWeights:
    """Oracle-format weights (``oracle.deepseek_port.gen_moe``: router (E, D),
    experts[e] = {gate (F, D), up (F, D), down (D, F)}, shared likewise or
    None) -> MoeWeights on the device."""
    import torch
    dev = device or _native.require_cuda()
    router = np.asarray(w["router"], np.float32)
    E, D = router.shape
    F = np.asarray(w["experts"][0]["gate"]).shape[0]

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).half()

    gu, dn = [], []
    for e in range(E):
        ex = w["experts"][e]
        if ex["gate"].shape != (F, D) or ex["up"].shape != (F, D) or ex["down"].shape != (D, F):
            raise ShapeMismatch(f"expert {e} shapes inconsistent with router {router.shape}")
        gu.append(gate_up_tiles(up(ex["gate"]), up(ex["up"])))
        dn.append(down_blocks(up(ex["down"])))
    sh = w.get("shared")
    mw = MoeWeights(D, E, top_k, F, 0 if sh is None else sh["gate"].shape[0], float(routed_scale),
                    up(router), torch.stack(gu).contiguous(), torch.stack(dn).contiguous())
    if sh is not None:
        mw.s_gu = gate_up_tiles(up(sh["gate"]), up(sh["up"]))
        mw.s_dn = down_blocks(up(sh["down"]))
    return mw


def random_moe_device(hidden: int, n_experts: int, inter: int, n_shared: int, top_k: int,
                      seed: int = 0, routed_scale: float = 1.0, device=None) -> MoeWeights:
    """Random fp16 MoE weights drawn directly on the device in the kernel
    layouts (benchmarks; same scales as the oracle generator)."""
    import torch
    dev = device or _native.require_cuda()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    D, E, F = hidden, n_experts, inter

    def rnd(shape, scale):
        return (torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * scale).half()

    Q = moe_segments(D)
    mw = MoeWeights(D, E, top_k, F, F * n_shared, float(routed_scale), rnd((E, D), D ** -0.5),
                    rnd((E, F // 2, D // 8, 4, 8), D ** -0.5),
                    rnd((E, F // 8, Q, 8, D // Q), F ** -0.5))
    if n_shared:
        Fs = F * n_shared
        mw.s_gu = rnd((Fs // 2, D // 8, 4, 8), D ** -0.5)
        mw.s_dn = rnd((Fs // 8, Q, 8, D // Q), Fs ** -0.5)
    return mw


class MoeWorkspace:
    """Per-stream workspace of the fused MoE launch (per-CTA partial sums,
    grid-barrier counter, routing outputs)."""

    def __init__(self, mw: MoeWeights, batch: int, device=None):
        import torch
        dev = device or _native.require_cuda()
        sms = max(int(_native.lib().cfb_device_sm_count()), 1)
        self.part = torch.zeros(sms, batch * mw.hidden, device=dev, dtype=torch.float32)
        self.barrier = torch.zeros(2, device=dev, dtype=torch.int64)  # grid barrier, route counter
        self.logits = torch.zeros(batch, mw.n_experts, device=dev, dtype=torch.float32)
        self.route_idx = torch.zeros(batch, mw.top_k, device=dev, dtype=torch.int32)
        self.route_w = torch.zeros(batch, mw.top_k, device=dev, dtype=torch.float32)
        torch.cuda.synchronize()  # zero counters visible to launches on any stream


def moe_launch(mw: MoeWeights, ws: MoeWorkspace, out, *, x=None, resid=None, norm_w=None,
               accum_in=None, eps: float = 1e-6, pdl: bool = False, grid: int = 0,
               stream=None, trace=None, partial: bool = False) -> None:
    """Enqueue one fused MoE launch (device tensors; no host sync).
    ``partial`` (tensor-parallel rank > 0): out = this rank's expert-shard
    partial instead of resid + attention + MoE."""
    B = out.shape[0]
    flags = (_native.NORM | _native.RESID) if resid is not None else 0
    if partial:
        flags |= _native.PARTIAL
    if pdl:
        flags |= _native.PDL
    a = _native.MoeArgs(
        dtype=2, batch=B, hidden=mw.hidden, n_experts=mw.n_experts, top_k=mw.top_k,
        inter=mw.inter, shared_inter=mw.shared_inter, flags=flags, grid=grid, eps=eps,
        routed_scale=mw.routed_scale, x=_native.ptr(x), resid=_native.ptr(resid),
        accum_in=_native.ptr(accum_in), norm_w=_native.ptr(norm_w), w_router=mw.router.data_ptr(),
        w_gu=mw.w_gu.data_ptr(), w_dn=mw.w_dn.data_ptr(), s_gu=_native.ptr(mw.s_gu),
        s_dn=_native.ptr(mw.s_dn), part=ws.part.data_ptr(), out=out.data_ptr(),
        route_idx=ws.route_idx.data_ptr(), route_w=ws.route_w.data_ptr(),
        barrier=ws.barrier.data_ptr(), logits=ws.logits.data_ptr(), trace=_native.ptr(trace))
    _native.check(_native.lib().cfb_moe_decode(a, _native.stream_ptr(stream)))


def run_moe_decode(h, w, top_k: int, routed_scale: float = 1.0, *, resid=None, norm_w=None,
                   eps: float = 1e-6, packed: MoeWeights | None = None, grid: int = 0):
    """MoE forward of B token rows on the GPU.

    ``h`` (B, D) fp16-valued activations, or - with ``resid``/``norm_w`` - the
    kernel computes h = f16(rmsnorm(resid) * norm_w) itself and returns
    resid + MoE(h) (the decoder-block form).  Returns (y (B, D) f32,
    expert ids (B, top_k) in selection order, gate weights (B, top_k))."""
    import torch
    dev = _native.require_cuda()
    mw = packed or pack_moe(w, top_k, routed_scale, dev)
    src = np.asarray(resid if resid is not None else h, np.float32)
    if src.ndim != 2 or src.shape[1] != mw.hidden:
        raise ShapeMismatch(f"activations {src.shape} do not match hidden {mw.hidden}")
    B = src.shape[0]
    if B > 4:
        raise DimensionError("the fused MoE kernel supports batch <= 4")
    ws = MoeWorkspace(mw, B, dev)
    out = torch.empty(B, mw.hidden, device=dev, dtype=torch.float32)
    with torch.no_grad():
        t = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
        if resid is not None:
            g = torch.from_numpy(np.ascontiguousarray(norm_w, np.float32)).to(dev).half()
            moe_launch(mw, ws, out, resid=t, norm_w=g, eps=eps, grid=grid)
        else:
            moe_launch(mw, ws, out, x=t.half(), eps=eps, grid=grid)
        torch.cuda.synchronize()
    return out.cpu().numpy(), ws.route_idx.cpu().numpy().astype(np.int64), ws.route_w.cpu().numpy()
