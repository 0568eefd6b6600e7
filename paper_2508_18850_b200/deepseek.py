"""DeepSeek-V2-Lite-shaped decoder block on the GPU (BASELINE.json config #3).

One block = the attention half then the MoE, chained with programmatic
dependent launch:

  1. MLA latent attention with the RMSNorm prologue x = f16(rmsnorm(resid) *
     g_attn), head sum into the 64-bit fixed-point accumulator.  At batch 1
     with the DeepSeek shape (16 heads, kv_lora_rank 512) this is the
     head-batched engine (``csrc/mla_engine.cu``: 3 launches, every weight and
     latent row read once); otherwise the reference-dataflow kernel
     (``csrc/attn_mla.cu``, ``run_fused_mla_decode``, ``dataflows.py:316-429``,
     CFB_NORM);
  2. fused MoE (``csrc/moe.cu``): r = resid + head sum, h = f16(rmsnorm(r) *
     g_ffn), router + softmax top-k, shared + routed SwiGLU experts,
     resid <- r + MoE(h).

Dims: the reference preset for MLA (hidden 2048, 16 heads x 128,
kv_lora_rank 512; ``cli.py:47-54``) and the DeepSeek-V2-Lite MoE (64 routed
experts, top-6, 2 shared, width 1408).  The CPU restatement is
``oracle/deepseek_port.block``.  The latent cache is an input (the reference
never appends to it, ``dataflows.py:393-397``): the new token's latent row is
attended once.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

from . import _native
from .exceptions import DimensionError
from .fused import padded_hidden, pow2_at_least
from .layouts import rotated_rows, row_tiles
from .mla import pack_mla
from .moe import MoeWeights, MoeWorkspace, moe_launch, pack_moe, random_moe_device


@dataclass(frozen=True)
class DeepSeekDims:
    hidden: int = 2048
    n_heads: int = 16
    head_dim: int = 128
    kv_rank: int = 512
    n_experts: int = 64
    top_k: int = 6
    inter: int = 1408
    n_shared: int = 2
    cluster: int = 4
    eps: float = 1e-6
    routed_scale: float = 1.0

    def mla_bytes(self, seq_len: int) -> int:
        """Algorithmic HBM bytes of the attention half: MLA weights + the
        latent cache read once + the norm gain (fp16)."""
        D, nh, H, R = self.hidden, self.n_heads, self.head_dim, self.kv_rank
        w = nh * D * H + D * R + nh * H * R + nh * R * H + nh * H * D
        return 2 * (w + seq_len * R + D)

    def moe_bytes(self) -> int:
        D = self.hidden
        return 2 * (self.n_experts * D + 3 * D * self.inter * (self.top_k + self.n_shared) + D)

    def block_bytes(self, seq_len: int) -> int:
        return self.mla_bytes(seq_len) + self.moe_bytes()


LITE = DeepSeekDims()


def engine_supported(dims: "DeepSeekDims", batch: int) -> bool:
    """The head-batched MLA engine (csrc/mla_engine.cu) covers the
    DeepSeek-V2-Lite/preset shape at batch 1; other shapes run the reference
    dataflow kernel (csrc/attn_mla.cu)."""
    return (batch == 1 and 1 <= dims.n_heads <= 16 and dims.kv_rank == 512 and dims.head_dim % 8 == 0
            and dims.head_dim <= 128 and dims.hidden % 512 == 0)


def pack_mla_engine(w_q, w_up, w_kv, w_down, w_out, cache, dev):
    """Reference MLA layouts (scenarios.py:140-165: w_q (nh, D, H), w_up
    (nh, H, R), w_kv (D, R), w_down (nh, R, H), w_out (nh, H, D), cache (S, R))
    -> cfb_mla_engine_args layouts (torch fp16 on `dev`)."""
    import torch

    def t(a):
        if isinstance(a, torch.Tensor):
            return a.to(dev).half()
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).half()

    wq, wup, wkv, wdn, wo = t(w_q), t(w_up), t(w_kv), t(w_down), t(w_out)
    nh, D, H = wq.shape
    R = wkv.shape[1]
    w_a = torch.cat([wq.permute(0, 2, 1).reshape(nh * H, D), wkv.t()], 0).contiguous()
    out = dict(w_a=row_tiles(w_a),
               w_up=rotated_rows(wup.permute(0, 2, 1).reshape(nh * R, H).contiguous()),
               w_dn=wdn.reshape(nh * R, H).contiguous(),
               w_o=row_tiles(wo.reshape(nh * H, D).t().contiguous()))
    S = cache.shape[0]
    out["cache"] = t(cache).contiguous() if S else torch.zeros(1, R, device=dev, dtype=torch.float16)
    out["S"] = S
    return out


class DeepSeekBlock:
    """Device-resident block: packed MLA + MoE weights, latent cache, norms,
    and the fixed-point workspaces.  ``launch(resid)`` updates ``resid``
    ([B][D] fp32, device) in place."""

    def __init__(self, dims: DeepSeekDims, mla: dict | None, moe: MoeWeights, attn_norm, ffn_norm,
                 seq_len: int, batch: int = 1, engine: dict | None = None):
        """`mla`: pack_mla layouts (reference-dataflow kernel) or None;
        `engine`: pack_mla_engine layouts (head-batched engine) or None -
        the engine is used when given."""
        import torch
        dev = _native.require_cuda()
        self.partial = False  # tensor-parallel rank > 0: the MoE writes its partial only
        if batch > 4:
            raise DimensionError("the DeepSeek block supports batch <= 4")
        if engine is None and (mla is None or mla["Dp"] != dims.hidden):
            raise DimensionError("the block's RMSNorm needs hidden % cluster == 0 and 16-byte rows")
        self.dims, self.mla, self.moe, self.S, self.B = dims, mla, moe, seq_len, batch
        self.engine = engine
        self.attn_norm, self.ffn_norm = attn_norm, ffn_norm
        self.accum_attn = torch.zeros(batch, dims.hidden, device=dev, dtype=torch.int64)
        self.ws = MoeWorkspace(moe, batch, dev)
        if engine is not None:
            nh, H, R = dims.n_heads, dims.head_dim, dims.kv_rank
            sms = max(int(_native.lib().cfb_device_sm_count()), 1)
            self.eng_ws = dict(
                qc=torch.zeros(nh * H + R, device=dev, dtype=torch.float16),
                qlat=torch.zeros(nh * R, device=dev, dtype=torch.float16),
                # partials keep all 16 MMA head rows whatever nh is (cfb.h)
                part=torch.zeros(sms, 2 * 16 + 16 * R, device=dev, dtype=torch.float32),
                o_acc=torch.zeros(nh * H, device=dev, dtype=torch.int64),
                barrier=torch.zeros(2, device=dev, dtype=torch.int64))
        # the workspaces were zeroed on torch's current stream; launches may use
        # another stream, and the monotonic counters must read zero there
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- builders
    @classmethod
    def from_arrays(cls, dims: DeepSeekDims, mla_arrays: dict, moe_w: dict, attn_norm, ffn_norm,
                    batch: int = 1, use_engine: bool = True) -> "DeepSeekBlock":
        """Oracle-format inputs: ``mla_arrays`` holds the reference MLA weights
        and cache (``w_q``, ``w_up``, ``w_kv``, ``w_down``, ``w_out``,
        ``kv_cache``; scenarios.py:140-165 layouts), ``moe_w`` the
        ``oracle.deepseek_port.gen_moe`` dict."""
        import torch
        dev = _native.require_cuda()
        S = mla_arrays["kv_cache"].shape[0]
        md = SimpleNamespace(batch_size=batch, hidden_dim=dims.hidden, n_heads=dims.n_heads,
                             head_dim=dims.head_dim, kv_lora_rank=dims.kv_rank, seq_len=S,
                             dtype_bytes=2)
        sc = SimpleNamespace(dims=md, cluster=SimpleNamespace(n_blocks=dims.cluster),
                             hidden=np.zeros((batch, dims.hidden), np.float32), **mla_arrays)
        if engine_supported(dims, batch) and use_engine:
            mla, eng = None, pack_mla_engine(*(mla_arrays[k] for k in ("w_q", "w_up", "w_kv", "w_down",
                                                                       "w_out", "kv_cache")), dev)
        else:
            mla, eng = pack_mla(sc, dev, torch.float16, cached=False), None
        moe = pack_moe(moe_w, dims.top_k, dims.routed_scale, dev)

        def g(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).half()

        return cls(dims, mla, moe, g(attn_norm), g(ffn_norm), S, batch, engine=eng)

    @classmethod
    def random(cls, dims: DeepSeekDims, seq_len: int, seed: int = 0, batch: int = 1,
               use_engine: bool = True) -> "DeepSeekBlock":
        """Random fp16 weights (scales of scenarios.py:155-162) and latent
        cache, drawn on the device."""
        import torch
        dev = _native.require_cuda()
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        D, nh, H, R = dims.hidden, dims.n_heads, dims.head_dim, dims.kv_rank

        def rnd(shape, scale):
            return torch.randn(*shape, generator=g, device=dev) * scale

        arrs = dict(w_q=rnd((nh, D, H), D ** -0.5), w_up=rnd((nh, H, R), H ** -0.5),
                    w_kv=rnd((D, R), D ** -0.5), w_down=rnd((nh, R, H), R ** -0.5),
                    w_out=rnd((nh, H, D), H ** -0.5), kv_cache=rnd((seq_len, R), 1.0))
        if engine_supported(dims, batch) and use_engine:
            mla, eng = None, pack_mla_engine(*(arrs[k] for k in ("w_q", "w_up", "w_kv", "w_down",
                                                                 "w_out", "kv_cache")), dev)
        else:
            md = SimpleNamespace(batch_size=batch, hidden_dim=D, n_heads=nh, head_dim=H,
                                 kv_lora_rank=R, seq_len=seq_len, dtype_bytes=2)
            sc = SimpleNamespace(dims=md, cluster=SimpleNamespace(n_blocks=dims.cluster),
                                 hidden=np.zeros((batch, D), np.float32),
                                 **{k: v.cpu().numpy() for k, v in arrs.items()})
            mla, eng = pack_mla(sc, dev, torch.float16, cached=False), None
        del arrs
        moe = random_moe_device(dims.hidden, dims.n_experts, dims.inter, dims.n_shared, dims.top_k,
                                seed=seed, routed_scale=dims.routed_scale, device=dev)
        ones = torch.ones(dims.hidden, device=dev, dtype=torch.float16)
        return cls(dims, mla, moe, ones, ones.clone(), seq_len, batch, engine=eng)

    # ---------------------------------------------------------------- launch
    def mla_args(self, resid, pdl: bool):
        d, pk = self.dims, self.mla
        flags = _native.APPEND | _native.NORM | (_native.PDL if pdl else 0)
        return _native.MlaArgs(
            dtype=2, batch=self.B, hidden=pk["Dp"], n_heads=d.n_heads, head_dim=d.head_dim,
            head_pad=pk["Hp"], kv_rank=d.kv_rank, rank_pad=pk["Rp"], cluster=d.cluster,
            seq_len=self.S, flags=flags, x=None, w_q=pk["w_q"].data_ptr(),
            w_kv=pk["w_kv"].data_ptr(), w_up=pk["w_up"].data_ptr(), w_down=pk["w_down"].data_ptr(),
            w_out=pk["w_out"].data_ptr(), cache=pk["cache"].data_ptr(), out=None,
            accum=self.accum_attn.data_ptr(), stats=None, traffic=None, resid=resid.data_ptr(),
            norm_w=self.attn_norm.data_ptr(), eps=d.eps)

    def engine_args(self, resid, pdl: bool):
        d, e, w = self.dims, self.engine, self.eng_ws
        return _native.MlaEngineArgs(
            hidden=d.hidden, n_heads=d.n_heads, head_dim=d.head_dim, kv_rank=d.kv_rank,
            seq_len=e["S"], flags=_native.PDL if pdl else 0, max_parts=w["part"].shape[0],
            eps=d.eps, resid=resid.data_ptr(), norm_w=self.attn_norm.data_ptr(),
            w_a=e["w_a"].data_ptr(), w_up=e["w_up"].data_ptr(), w_dn=e["w_dn"].data_ptr(),
            w_o=e["w_o"].data_ptr(), cache=e["cache"].data_ptr(), qc=w["qc"].data_ptr(),
            qlat=w["qlat"].data_ptr(), part=w["part"].data_ptr(),
            o_acc=w["o_acc"].data_ptr(), accum=self.accum_attn.data_ptr(),
            barrier=w["barrier"].data_ptr(),
            trace=self.trace.data_ptr() if getattr(self, "trace", None) is not None else None)

    def launch_attention(self, resid, pdl: bool = True, stream=None) -> None:
        if self.engine is not None:
            _native.check(_native.lib().cfb_mla_engine_decode(self.engine_args(resid, pdl),
                                                              _native.stream_ptr(stream)))
        else:
            _native.check(_native.lib().cfb_mla_decode(self.mla_args(resid, pdl),
                                                       _native.stream_ptr(stream)))

    def launch(self, resid, pdl: bool = True, stream=None, attn_reduce=None) -> None:
        """Enqueue the block on `stream`: resid <- block(resid).  Tensor
        parallel (tp.TPDeepSeekBlock): ``attn_reduce(accum_attn)`` sums the
        ranks' fixed-point attention partials between the halves."""
        self.launch_attention(resid, pdl, stream)
        if attn_reduce is not None:
            attn_reduce(self.accum_attn)
        moe_launch(self.moe, self.ws, resid, resid=resid, norm_w=self.ffn_norm,
                   accum_in=self.accum_attn, eps=self.dims.eps, pdl=pdl and attn_reduce is None,
                   stream=stream, partial=self.partial, trace=getattr(self, "moe_trace", None))

    def run(self, resid_host) -> tuple[np.ndarray, np.ndarray]:
        """Host convenience: one block on (B, D) fp32 rows.  Returns (new
        residual rows, routed expert ids in selection order)."""
        import torch
        dev = _native.require_cuda()
        r = torch.from_numpy(np.ascontiguousarray(resid_host, np.float32)).to(dev)
        self.launch(r, pdl=False)
        torch.cuda.synchronize()
        return r.cpu().numpy(), self.ws.route_idx.cpu().numpy().astype(np.int64)


def mla_padding_ok(dims: DeepSeekDims) -> bool:
    return padded_hidden(dims.hidden, dims.cluster, 2) == dims.hidden and \
        pow2_at_least(dims.head_dim) >= dims.head_dim
