"""ctypes binding of ``libcfb.so`` (the C ABI declared in ``include/cfb.h``).

The library is built in-tree by ``__graft_entry__.build()`` (``make`` in
``csrc/``).  There is no fallback: if the library or a CUDA device is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .exceptions import (DimensionError, InvalidClusterSize, ShapeMismatch, SimulationError,
                         SmemOverflow)

LIB_PATH = Path(__file__).resolve().parent / "libcfb.so"

CFB_F16, CFB_F32 = 2, 4
APPEND, WRITE_KV, ROPE, NORM, RESID, STATS_MERGED, PDL, ONESHOT = 1, 2, 4, 8, 16, 32, 64, 128
PARTIAL, DYN_POOL, TC_PAIR = 256, 1024, 2048
STAGE_NAMES = ("qkv_gather", "stats_max_reduce", "stats_sum_reduce", "stats_merge_reduce",
               "attn_out_reduce", "q_proj_gather", "latent_kv_gather", "absorbed_q_gather",
               "down_proj_reduce", "score_reduce", "out_proj_reduce")

_vp = ctypes.c_void_p


class MhaArgs(ctypes.Structure):
    """Mirror of ``cfb_mha_args``."""

    _fields_ = [
        ("dtype", ctypes.c_int), ("batch", ctypes.c_int), ("hidden", ctypes.c_int),
        ("n_heads", ctypes.c_int), ("head_dim", ctypes.c_int), ("head_pad", ctypes.c_int),
        ("cluster", ctypes.c_int), ("seq_len", ctypes.c_int), ("cache_cap", ctypes.c_int),
        ("flags", ctypes.c_int),
        ("x", _vp), ("resid", _vp), ("norm_w", _vp), ("eps", ctypes.c_float),
        ("w_qkv", _vp), ("w_out", _vp), ("k_cache", _vp), ("v_cache", _vp),
        ("rope_cs", _vp), ("step_pos", _vp), ("out", _vp), ("accum", _vp),
        ("stats", _vp), ("traffic", _vp), ("trace", _vp),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcfb.so once; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise SimulationError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
        L.cfb_mha_decode.argtypes = [ctypes.POINTER(MhaArgs), _vp]
        L.cfb_mha_decode.restype = ctypes.c_int
        L.cfb_cluster_collective.argtypes = [ctypes.c_int] * 4 + [_vp, _vp, _vp, _vp]
        L.cfb_cluster_collective.restype = ctypes.c_int
        L.cfb_last_error.restype = ctypes.c_char_p
        L.cfb_version.restype = ctypes.c_char_p
        L.cfb_device_sm_count.restype = ctypes.c_int
        bind_extra(L)
        _lib = L
    return _lib


_STATUS = {-1: DimensionError, -2: InvalidClusterSize, -3: ShapeMismatch, -4: SmemOverflow,
           -5: SimulationError, -6: ValueError}


def check(status: int) -> None:
    """Translate a cfb_status into the reference's exception classes."""
    if status != 0:
        msg = lib().cfb_last_error().decode(errors="replace")
        raise _STATUS.get(status, SimulationError)(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise SimulationError("paper_2508_18850_b200 needs a CUDA (sm_100a) device; "
                              "there is no CPU fallback")
    return torch.device("cuda")


class MlaArgs(ctypes.Structure):
    """Mirror of ``cfb_mla_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "batch", "hidden", "n_heads", "head_dim",
                                             "head_pad", "kv_rank", "rank_pad", "cluster",
                                             "seq_len", "flags")] + [
        (n, _vp) for n in ("x", "w_q", "w_kv", "w_up", "w_down", "w_out", "cache", "out", "accum",
                           "stats", "traffic", "resid", "norm_w")] + [("eps", ctypes.c_float)]


class SplitHeadArgs(ctypes.Structure):
    """Mirror of ``cfb_splithead_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "batch", "hidden", "n_heads", "head_dim",
                                             "cluster", "seq_len", "flags")] + [
        (n, _vp) for n in ("x", "w_qkv", "w_out", "k_cache", "v_cache", "out", "accum", "stats",
                           "traffic")]


class FfnArgs(ctypes.Structure):
    """Mirror of ``cfb_ffn_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "batch", "hidden", "inter", "flags", "grid")] + [
        ("eps", ctypes.c_float), ("x", _vp), ("resid", _vp), ("accum", _vp), ("norm_w", _vp), ("w_gu", _vp),
        ("w_dn", _vp), ("act", _vp), ("out", _vp), ("barrier", _vp), ("trace", _vp)]


class LmArgs(ctypes.Structure):
    """Mirror of ``cfb_lm_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "batch", "hidden", "vocab", "grid", "flags")] + [
        ("eps", ctypes.c_float), ("resid", _vp), ("norm_w", _vp), ("w", _vp), ("logits", _vp),
        ("cand_val", _vp), ("cand_idx", _vp), ("ticket", _vp), ("token_out", _vp),
        ("step_pos", _vp)]


class MlaEngineArgs(ctypes.Structure):
    """Mirror of ``cfb_mla_engine_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("hidden", "n_heads", "head_dim", "kv_rank", "seq_len",
                                             "flags", "max_parts")] + [
        ("eps", ctypes.c_float)] + [
        (n, _vp) for n in ("resid", "norm_w", "w_a", "w_up", "w_dn", "w_o", "cache", "qc", "qlat",
                           "part", "o_acc", "accum", "barrier", "trace")]


class FfnB16Args(ctypes.Structure):
    """Mirror of ``cfb_ffn_b16_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("hidden", "inter", "flags")] + [("eps", ctypes.c_float)] + [
        (n, _vp) for n in ("resid", "norm_w", "w_gu", "w_dn", "xp", "gu_acc", "ap", "out_acc", "ticket")] + [
        ("batch", ctypes.c_int), ("slots", _vp)]


class B16LayerArgs(ctypes.Structure):
    """Mirror of ``cfb_b16_layer_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("hidden", "n_heads", "inter", "cache_cap", "max_len",
                                             "flags", "stage")] + [("eps", ctypes.c_float)] + [
        (n, _vp) for n in ("resid", "attn_norm", "ffn_norm", "w_qkv", "w_o", "w_gu", "w_dn", "k_cache",
                           "v_cache", "rope_cs", "pos", "xp", "q16", "qkv_acc", "part", "o_acc",
                           "gu_acc", "ap", "ticket", "block_table")] + [("max_pages", ctypes.c_int),
                                                                        ("batch", ctypes.c_int),
                                                                        ("slots", _vp)]


class MoeArgs(ctypes.Structure):
    """Mirror of ``cfb_moe_args``."""

    _fields_ = [(n, ctypes.c_int) for n in ("dtype", "batch", "hidden", "n_experts", "top_k",
                                             "inter", "shared_inter", "flags", "grid")] + [
        ("eps", ctypes.c_float), ("routed_scale", ctypes.c_float)] + [
        (n, _vp) for n in ("x", "resid", "accum_in", "norm_w", "w_router", "w_gu", "w_dn", "s_gu",
                           "s_dn", "part", "out", "route_idx", "route_w", "barrier", "logits", "trace")]


def bind_extra(L) -> None:
    L.cfb_collective_bench.argtypes = [ctypes.c_int] * 6 + [_vp] * 6
    L.cfb_collective_bench.restype = ctypes.c_int
    L.cfb_tc_gemm_b16.argtypes = [_vp] * 6 + [ctypes.c_int] * 3 + [_vp]
    L.cfb_tc_gemm_b16.restype = ctypes.c_int
    L.cfb_ffn_b16.argtypes = [ctypes.POINTER(FfnB16Args), _vp]
    L.cfb_b16_slots_floats.argtypes = [ctypes.c_int] * 4
    L.cfb_b16_slots_floats.restype = ctypes.c_size_t
    L.cfb_ffn_b16.restype = ctypes.c_int
    L.cfb_llama_b16_layer.argtypes = [ctypes.POINTER(B16LayerArgs), _vp]
    L.cfb_llama_b16_layer.restype = ctypes.c_int
    L.cfb_b16_advance.argtypes = [_vp, ctypes.c_int, _vp]
    L.cfb_b16_advance.restype = ctypes.c_int
    L.cfb_b16_lm_head.argtypes = [_vp] * 3 + [ctypes.c_int] * 2 + [ctypes.c_float] + [_vp] * 5 + [ctypes.c_int, _vp]
    L.cfb_b16_lm_head.restype = ctypes.c_int
    L.cfb_b16_kv_write.argtypes = [_vp] * 3 + [ctypes.c_int] * 6 + [_vp] * 3
    L.cfb_b16_kv_write.restype = ctypes.c_int
    L.cfb_embed.argtypes = [ctypes.c_int] + [_vp] * 3 + [ctypes.c_int] * 2 + [_vp]
    L.cfb_embed.restype = ctypes.c_int
    L.cfb_mla_engine_decode.argtypes = [ctypes.POINTER(MlaEngineArgs), _vp]
    L.cfb_mla_engine_decode.restype = ctypes.c_int
    L.cfb_moe_decode.argtypes = [ctypes.POINTER(MoeArgs), _vp]
    L.cfb_moe_decode.restype = ctypes.c_int
    L.cfb_mla_decode.argtypes = [ctypes.POINTER(MlaArgs), _vp]
    L.cfb_mla_decode.restype = ctypes.c_int
    L.cfb_splithead_decode.argtypes = [ctypes.POINTER(SplitHeadArgs), _vp]
    L.cfb_splithead_decode.restype = ctypes.c_int
    L.cfb_ffn_decode.argtypes = [ctypes.POINTER(FfnArgs), _vp]
    L.cfb_ffn_decode.restype = ctypes.c_int
    L.cfb_lm_head_argmax.argtypes = [ctypes.POINTER(LmArgs), _vp]
    L.cfb_lm_head_argmax.restype = ctypes.c_int
