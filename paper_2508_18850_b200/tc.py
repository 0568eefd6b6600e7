"""Batch-16 projections on the tcgen05 tensor cores (``csrc/tc_gemm.cu``).

y[n][m] = sum_k W[m][k] x[n][k] for 16 batch rows: the weights are the MMA's
M = 128 operand (swap-AB), accumulators live in TMEM, split-K partials are
summed in 64-bit fixed point.  ``pack_umma`` lays W out in the UMMA K-major
no-swizzle core-matrix order so the kernel's plain bulk copies land in the
canonical shared-memory layout.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .exceptions import DimensionError

BATCH = 16


def pack_umma(w):
    """(M, K) fp16 torch tensor -> [M/128][K/64][4][2][16][8][8] (flattened)."""
    M, K = w.shape
    if M % 128 or K % 64:
        raise DimensionError("tcgen05 projection needs M % 128 == 0 and K % 64 == 0")
    t = w.reshape(M // 128, 16, 8, K // 64, 4, 2, 8)      # (t, g, r, kb, s, c, e)
    return t.permute(0, 3, 4, 5, 1, 2, 6).contiguous()


class TcProjection:
    """Device-resident packed weight + workspaces for y = x W^T at batch 16."""

    def __init__(self, w, device=None):
        import torch
        dev = device or _native.require_cuda()
        if not isinstance(w, torch.Tensor):
            w = torch.from_numpy(np.ascontiguousarray(w, np.float32))
        w = w.to(dev).half()
        self.M, self.K = w.shape
        self.wp = pack_umma(w)
        self.xp = torch.zeros(BATCH * self.K, device=dev, dtype=torch.float16)
        self.acc = torch.zeros(BATCH, self.M, device=dev, dtype=torch.int64)
        torch.cuda.synchronize()

    def launch(self, x, y=None, resid=None, pdl=False, stream=None, pair=False):
        """x: (16, K) fp16 device tensor; y: (16, M) fp32 or None (sum stays in acc);
        pair: CTA pairs sharing each activation block by TMA multicast."""
        _native.check(_native.lib().cfb_tc_gemm_b16(
            self.wp.data_ptr(), x.data_ptr(), self.xp.data_ptr(), self.acc.data_ptr(),
            _native.ptr(y), _native.ptr(resid), self.M, self.K,
            (_native.PDL if pdl else 0) | (_native.TC_PAIR if pair else 0), _native.stream_ptr(stream)))


def run_projection_b16(w, x, pair: bool = False) -> np.ndarray:
    """Host convenience: (M, K) weights, (16, K) activations -> (16, M) fp32."""
    import torch
    dev = _native.require_cuda()
    proj = TcProjection(w, dev)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev).half()
    if xt.shape != (BATCH, proj.K):
        raise DimensionError(f"x must be ({BATCH}, {proj.K})")
    y = torch.empty(BATCH, proj.M, device=dev, dtype=torch.float32)
    proj.launch(xt, y, pair=pair)
    torch.cuda.synchronize()
    return y.cpu().numpy()


class TcFfnB16:
    """Batch-16 SwiGLU FFN block on tcgen05 (``cfb_ffn_b16``): resid += FFN(rmsnorm(resid))."""

    def __init__(self, w1, w2, w3, norm_w, eps: float = 1e-5, device=None):
        import torch
        dev = device or _native.require_cuda()

        def t(a):
            if not isinstance(a, torch.Tensor):
                a = torch.from_numpy(np.ascontiguousarray(a, np.float32))
            return a.to(dev).half()

        w1, w2, w3 = t(w1), t(w2), t(w3)
        self.F, self.D = w1.shape
        self.eps = eps
        # gate/up rows interleaved per 64 (one 128-row tile = 64 gate + their 64 up rows)
        self.w_gu = pack_umma(torch.stack([w1.reshape(-1, 64, self.D), w2.reshape(-1, 64, self.D)], 1)
                              .reshape(2 * self.F, self.D))
        self.w_dn = pack_umma(w3)
        self.g = t(norm_w)
        self.xp = torch.zeros(BATCH * self.D, device=dev, dtype=torch.float16)
        self.gu_acc = torch.zeros(BATCH * 2 * self.F, device=dev, dtype=torch.int64)
        self.ap = torch.zeros(BATCH * self.F, device=dev, dtype=torch.float16)
        self.out_acc = torch.zeros(BATCH * self.D, device=dev, dtype=torch.int64)
        self.ticket = torch.zeros((2 * self.F + self.D) // 128, device=dev, dtype=torch.int32)
        self.slots = torch.zeros(int(_native.lib().cfb_b16_slots_floats(self.D, 0, self.F, BATCH)),
                                 device=dev, dtype=torch.float32)
        torch.cuda.synchronize()

    @property
    def weight_bytes(self) -> int:
        return 3 * self.D * self.F * 2 + self.D * 2

    def launch(self, resid, pdl: bool = False, stream=None, pair: bool = False) -> None:
        a = _native.FfnB16Args(hidden=self.D, inter=self.F,
                               flags=(_native.PDL if pdl else 0) | (_native.TC_PAIR if pair else 0),
                               eps=self.eps, resid=resid.data_ptr(), norm_w=self.g.data_ptr(),
                               w_gu=self.w_gu.data_ptr(), w_dn=self.w_dn.data_ptr(),
                               xp=self.xp.data_ptr(), gu_acc=self.gu_acc.data_ptr(),
                               ap=self.ap.data_ptr(), out_acc=self.out_acc.data_ptr(),
                               ticket=self.ticket.data_ptr(), batch=BATCH, slots=self.slots.data_ptr())
        _native.check(_native.lib().cfb_ffn_b16(a, _native.stream_ptr(stream)))
