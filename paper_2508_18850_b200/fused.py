"""Drop-in fused decode dataflows backed by the sm_100a kernels in libcfb.so.

Same names, arguments, results and errors as the reference's
``dataflows.py`` (``run_fused_mha_decode`` :235-313, ``run_dataflow``
:505-514, ``DecodeResult`` :55-68).  The numerics run on the GPU: the
scenario's arrays are packed once per call into the kernels' HBM layouts
(fp16 when ``dtype_bytes == 2``), the kernel is launched through the C ABI,
and the result carries the device output plus the DSMEM ledger of the
kernel's static collective schedule, cross-checked against the byte counters
the kernel itself kept.

Deliberate, documented deviation: heads are summed in
64-bit fixed point (value x 2^32, integer atomics: exact and order-free)
instead of the reference's f16-rounded atomic accumulation, so ``output`` is
closer to the dense fp32 oracle than the reference simulator's own f16
output, and bit-identical from run to run.
"""

from __future__ import annotations

import functools

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .exceptions import DimensionError, SimulationError
from .ledger import (GLOBAL, ONESHOT_MERGE, StageTrace, TrafficLedger, emit_gather, emit_oneshot,
                     emit_reduce)
from .layouts import gate_up_tiles, qkv_tiles, row_tiles, wo_rows
from .scenario import MHA, MLA, validate_scenario

SPLIT_TOKEN, FUSED_MLA, SPLIT_HEAD = "split_token", "fused_mla", "split_head"
DATAFLOW_KINDS = (SPLIT_TOKEN, FUSED_MLA, SPLIT_HEAD)
# "oneshot" extends the reference's stats modes (dataflows.py:187-227): the
# decode engine's single-round all-to-all gather + one fused fp32 (m, l, A)
# softmax-merge in place of the stats and attn_out reduces (CFB_ONESHOT).
TWO_PASS, MERGED, ONESHOT = "two_pass", "merged", "oneshot"


@dataclass
class DecodeResult:
    output: np.ndarray
    ledger: TrafficLedger
    stage_traffic: dict
    score_max: np.ndarray
    score_sum: np.ndarray
    collectives: list = field(default_factory=list)
    n_clusters: int = 0
    n_blocks: int = 1
    device_traffic: dict = field(default_factory=dict)  # bytes the kernel counted

    @property
    def dsmem_bytes(self) -> int:
        return self.ledger.channel_bytes("dsmem")


def sequence_segments(seq_len: int, n_blocks: int) -> list[tuple[int, int]]:
    """Contiguous ceil(S/N) KV segments per CTA (dataflows.py:109-114)."""
    if seq_len == 0:
        return [(0, 0)] * n_blocks
    step = -(-seq_len // n_blocks)
    return [(min(b * step, seq_len), min((b + 1) * step, seq_len)) for b in range(n_blocks)]


def validate_partitioning(scenario, kind: str, append_new_token: bool = True) -> None:
    """Partitioning rules and error types of dataflows.py:117-137."""
    n = scenario.cluster.n_blocks
    d = scenario.dims
    if kind not in DATAFLOW_KINDS:
        raise DimensionError(f"unknown dataflow kind {kind!r}")
    if d.seq_len == 0 and not append_new_token:
        raise DimensionError("no attended positions: empty cache and no appended token")
    if d.head_dim % n:
        raise DimensionError(f"head_dim {d.head_dim} not divisible by cluster size {n}")
    if kind in (SPLIT_TOKEN, FUSED_MLA) and d.hidden_dim % n:
        raise DimensionError(f"hidden_dim {d.hidden_dim} not divisible by cluster size {n}")
    if kind == FUSED_MLA:
        if scenario.kind != MLA:
            raise DimensionError("fused_mla requires an mla scenario")
        if d.kv_lora_rank is None or d.kv_lora_rank % n:
            raise DimensionError(f"kv_lora_rank {d.kv_lora_rank} not divisible by cluster size {n}")
    elif scenario.kind != MHA:
        raise DimensionError(f"{kind} requires an mha scenario")


def pow2_at_least(x: int, lo: int = 8) -> int:
    p = lo
    while p < x:
        p *= 2
    return p


def padded_hidden(D: int, n: int, dtype_bytes: int) -> int:
    """Smallest D' >= D with 16-byte rows and D' % n == 0 (zero padding)."""
    q = max(n, 16 // dtype_bytes)
    return -(-D // q) * q


def _emit_global(ledger, n, batch, out_slice, nbytes):
    for b in range(n):
        for _ in range(batch):
            ledger.record(-1, b, -1, out_slice * nbytes, GLOBAL)


def _finish_output(out: np.ndarray) -> np.ndarray:
    if not np.all(np.isfinite(out)):
        raise SimulationError("decode produced a non-finite output")
    return out


def _pack_mha_static(scenario, cached: bool = True) -> dict:
    """Packed device copies of the scenario's weights and KV cache (the
    per-call state is only the hidden vector): through the DeviceCache
    (checksum-validated) or freshly built for ``prepare``."""
    import torch
    from .devcache import CACHE
    dev = _native.require_cuda()
    d = scenario.dims
    n, nb = scenario.cluster.n_blocks, d.dtype_bytes
    D, nh, H, S = d.hidden_dim, d.n_heads, d.head_dim, d.seq_len
    dt = torch.float16 if nb == 2 else torch.float32
    Hp = pow2_at_least(H)
    Dp = padded_hidden(D, n, nb)

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)

    def get(arr, tag, build):
        return CACHE.get(arr, tag, build) if cached else build(arr)

    def b_qkv(a):  # w_qkv (nh, D, 3H) -> row tiles [head][rank][q|k|v slice][D']
        return qkv_tiles(up(a).to(dt), n, Hp, Dp)

    def b_wo(a):
        wo = torch.zeros(nh, Dp, Hp, device=dev, dtype=dt)
        wo[:, :D, :H] = up(a).transpose(1, 2).to(dt)
        return wo_rows(wo, n)

    def b_cache(a):
        c = torch.zeros(nh, max(S, 1), Hp, device=dev, dtype=dt)
        if S:
            c[:, :S, :H] = up(a).to(dt)
        return c

    with torch.no_grad():
        return dict(w_qkv=get(scenario.w_qkv, ("mha_qkv", n, Hp, Dp, nb), b_qkv),
                    w_out=get(scenario.w_out, ("mha_wo", n, Hp, Dp, nb), b_wo),
                    k_cache=get(scenario.k_cache, ("mha_kv", Hp, nb, S), b_cache),
                    v_cache=get(scenario.v_cache, ("mha_kv", Hp, nb, S), b_cache),
                    Hp=Hp, Dp=Dp, cap=max(S, 1))


@functools.lru_cache(maxsize=64)
def _mha_schedule_cached(nh, n, B, D, H, nb, stats_mode):
    """The static collective schedule of one split_token launch, emitted in
    the reference's event order (pure function of the shapes: memoised, the
    ~1,300 events of a Llama-dims call cost ~1 ms of Python to build)."""
    ledger = TrafficLedger()
    stage_traffic: dict[str, int] = {}
    traces = []
    h = H // n
    for head in range(nh):
        if stats_mode == ONESHOT:
            tr = [("qkv_gather", emit_oneshot(ledger, n, B * 3 * h * nb, "gather")),
                  ("attn_state_merge", emit_oneshot(ledger, n, (2 * B + B * H) * 4, ONESHOT_MERGE))]
        else:
            tr = [("qkv_gather", emit_gather(ledger, n, B * 3 * h * nb))]
        if stats_mode == ONESHOT:
            pass  # statistics travel inside attn_state_merge
        elif stats_mode == MERGED:
            tr.append(("stats_merge_reduce", emit_reduce(ledger, n, 2 * B * nb)))
        else:
            tr.append(("stats_max_reduce", emit_reduce(ledger, n, B * nb)))
            tr.append(("stats_sum_reduce", emit_reduce(ledger, n, B * nb)))
        if stats_mode != ONESHOT:
            tr.append(("attn_out_reduce", emit_reduce(ledger, n, B * H * nb)))
        for stage, t in tr:
            stage_traffic[stage] = stage_traffic.get(stage, 0) + t.dsmem_bytes
            traces.append(StageTrace(stage, head, t))
        _emit_global(ledger, n, B, D // n, nb)
    return tuple(ledger.events), tuple(stage_traffic.items()), tuple(traces)


def _mha_schedule(nh, n, B, D, H, nb, stats_mode):
    """Fresh (ledger, stage_traffic, traces) per call: the events and traces
    are immutable, the containers are new, so callers may extend them."""
    ev, st, tr = _mha_schedule_cached(nh, n, B, D, H, nb, stats_mode)
    ledger = TrafficLedger()
    ledger.events = list(ev)
    return ledger, dict(st), list(tr)


def run_fused_mha_decode(scenario, stats_mode: str = TWO_PASS,
                         append_new_token: bool = True) -> DecodeResult:
    """split_token fused attention module on the GPU (one cluster per head).

    ``scenario`` is a ``DecodeScenario`` (packed weights come from the
    checksum-validated device cache) or the ``PreparedScenario`` of
    ``prepare(scenario)`` (device-resident, no per-call re-validation)."""
    import torch
    from .devcache import PreparedScenario

    prepared = scenario if isinstance(scenario, PreparedScenario) else None
    if prepared is not None:
        scenario = prepared.scenario
    validate_partitioning(scenario, SPLIT_TOKEN, append_new_token)
    validate_scenario(scenario)
    if stats_mode not in (TWO_PASS, MERGED, ONESHOT):
        raise ValueError(f"unknown stats_mode {stats_mode!r}")
    dev = _native.require_cuda()
    d = scenario.dims
    n, nb = scenario.cluster.n_blocks, d.dtype_bytes
    B, D, nh, H, S = d.batch_size, d.hidden_dim, d.n_heads, d.head_dim, d.seq_len
    dt = torch.float16 if nb == 2 else torch.float32
    pk = prepared.packed if prepared is not None else _pack_mha_static(scenario)
    Hp, Dp, cap = pk["Hp"], pk["Dp"], pk["cap"]

    with torch.no_grad():
        x = torch.zeros(B, Dp, device=dev, dtype=dt)
        x[:, :D] = torch.from_numpy(np.ascontiguousarray(scenario.hidden, np.float32)).to(dev).to(dt)
        out = torch.empty(B, Dp, device=dev, dtype=torch.float32)
        L = _native.lib()
        accum = torch.zeros(B, Dp, device=dev, dtype=torch.int64)
        stats = torch.zeros(nh, 2, B, device=dev, dtype=torch.float32)
        traffic = torch.zeros(16, device=dev, dtype=torch.int64)
        flags = (_native.APPEND if append_new_token else 0) | {
            TWO_PASS: 0, MERGED: _native.STATS_MERGED, ONESHOT: _native.ONESHOT}[stats_mode]
        args = _native.MhaArgs(
            dtype=nb, batch=B, hidden=Dp, n_heads=nh, head_dim=H, head_pad=Hp, cluster=n,
            seq_len=S, cache_cap=cap, flags=flags, x=x.data_ptr(), eps=0.0,
            w_qkv=pk["w_qkv"].data_ptr(), w_out=pk["w_out"].data_ptr(), k_cache=pk["k_cache"].data_ptr(),
            v_cache=pk["v_cache"].data_ptr(), out=out.data_ptr(), accum=accum.data_ptr(),
            stats=stats.data_ptr(), traffic=traffic.data_ptr())
        _native.check(L.cfb_mha_decode(args, _native.stream_ptr()))
        torch.cuda.synchronize()
        out_np = out[:, :D].cpu().numpy()
        st = stats.cpu().numpy()
        dev_traffic = traffic.cpu().numpy()

    ledger, stage_traffic, traces = _mha_schedule(nh, n, B, D, H, nb, stats_mode)
    names = ["qkv_gather"] + (["stats_merge_reduce"] if stats_mode == MERGED
                              else ["stats_max_reduce", "stats_sum_reduce"]) + ["attn_out_reduce"]
    if stats_mode == ONESHOT:
        device_traffic = {"qkv_gather": int(dev_traffic[0]), "attn_state_merge": int(dev_traffic[4])}
    else:
        device_traffic = {_native.STAGE_NAMES[i]: int(dev_traffic[i]) for i in range(5)
                          if _native.STAGE_NAMES[i] in names}
    if device_traffic != stage_traffic:
        raise SimulationError(f"kernel DSMEM byte counters {device_traffic} disagree with the "
                              f"schedule {stage_traffic}")
    return DecodeResult(output=_finish_output(out_np), ledger=ledger, stage_traffic=stage_traffic,
                        score_max=np.ascontiguousarray(st[:, 0, :]),
                        score_sum=np.ascontiguousarray(st[:, 1, :]), collectives=traces,
                        n_clusters=nh, n_blocks=n, device_traffic=device_traffic)


def run_dataflow(kind: str, scenario, **kwargs) -> DecodeResult:
    """Dispatch by dataflow kind (dataflows.py:505-514)."""
    if kind == SPLIT_TOKEN:
        return run_fused_mha_decode(scenario, **kwargs)
    if kind == FUSED_MLA:
        from .mla import run_fused_mla_decode
        return run_fused_mla_decode(scenario, **kwargs)
    if kind == SPLIT_HEAD:
        from .mla import run_splithead_decode
        kwargs.pop("stats_mode", None)
        return run_splithead_decode(scenario, **kwargs)
    raise DimensionError(f"unknown dataflow kind {kind!r}")


def cluster_collective(payloads: np.ndarray, op: str, dtype_bytes: int = 4):
    """Run one DSMEM ClusterReduce ("sum"/"max"/"softmax_merge") or
    ClusterGather ("gather") on the GPU.  payloads: (N, n).  Returns
    (per-CTA buffers, dsmem bytes counted by the kernel)."""
    import torch
    dev = _native.require_cuda()
    ops = {"sum": 0, "max": 1, "softmax_merge": 2, "softmax-merge": 2, "gather": 3}
    if op not in ops:
        raise ValueError(f"unknown collective {op!r}")
    p = np.ascontiguousarray(payloads, dtype=np.float32)
    N, n = p.shape
    dt = torch.float16 if dtype_bytes == 2 else torch.float32
    inp = torch.from_numpy(p).to(dev).to(dt)
    out = torch.zeros((N, N * n) if op == "gather" else (N, n), device=dev, dtype=dt)
    traffic = torch.zeros(1, device=dev, dtype=torch.int64)
    _native.check(_native.lib().cfb_cluster_collective(dtype_bytes, ops[op], N, n, inp.data_ptr(),
                                                       out.data_ptr(), traffic.data_ptr(),
                                                       _native.stream_ptr()))
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), int(traffic.item())


def run_fused_ffn(z, w1, w2, w3, activation: str = "silu", dtype_bytes: int = 2,
                  resid=None, norm_w=None, eps: float = 1e-5) -> np.ndarray:
    """Fused gate/up -> SiLU*mul -> down in one launch; the reference's
    ``ffn_reference(z, w1, w2, w3, "silu")`` (oracle.py:112-131).

    With ``resid``/``norm_w`` the kernel computes z = f16(rmsnorm(resid)*norm_w)
    itself and returns resid + FFN(z) (the decoder-block form).  The
    activation vector is stored at ``dtype_bytes`` precision between the two
    GEMVs (it crosses CTAs through HBM)."""
    import torch
    if activation != "silu":
        raise DimensionError("the fused FFN kernel implements the SwiGLU ('silu') gate only")
    dev = _native.require_cuda()
    w1, w2, w3 = (np.asarray(a, np.float32) for a in (w1, w2, w3))
    F, D = w1.shape
    if w2.shape != (F, D) or w3.shape != (D, F):
        from .exceptions import ShapeMismatch
        raise ShapeMismatch(f"ffn shapes inconsistent: w1 {w1.shape}, w2 {w2.shape}, w3 {w3.shape}")
    dt = torch.float16 if dtype_bytes == 2 else torch.float32

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).to(dt)

    flags = 0
    B = (np.asarray(resid) if resid is not None else np.asarray(z)).shape[0]
    x = up(z) if resid is None else None
    r = torch.from_numpy(np.ascontiguousarray(resid, np.float32)).to(dev) if resid is not None else None
    g = up(norm_w) if norm_w is not None else None
    if resid is not None:
        flags |= _native.NORM | _native.RESID
    if F % 2 or D % 4:
        raise DimensionError("fused FFN needs an even intermediate size and hidden % 4 == 0")
    w_gu = gate_up_tiles(up(w1), up(w2))
    w_dn = row_tiles(up(w3))
    act = torch.empty(B, F, device=dev, dtype=dt)
    out = torch.empty(B, D, device=dev, dtype=torch.float32)
    bar = torch.zeros(1, device=dev, dtype=torch.int64)
    a = _native.FfnArgs(dtype=dtype_bytes, batch=B, hidden=D, inter=F, flags=flags, grid=0,
                        eps=eps, x=_native.ptr(x), resid=_native.ptr(r), norm_w=_native.ptr(g),
                        w_gu=w_gu.data_ptr(), w_dn=w_dn.data_ptr(), act=act.data_ptr(),
                        out=out.data_ptr(), barrier=bar.data_ptr())
    _native.check(_native.lib().cfb_ffn_decode(a, _native.stream_ptr()))
    return out.cpu().numpy()


def lm_head_argmax(resid, norm_w, w_lm, eps: float = 1e-5, dtype_bytes: int = 2):
    """Final RMSNorm + LM head + greedy argmax on the GPU.  Returns
    (logits (B, V) fp32, tokens (B,))."""
    import torch
    dev = _native.require_cuda()
    dt = torch.float16 if dtype_bytes == 2 else torch.float32
    r = torch.from_numpy(np.ascontiguousarray(resid, np.float32)).to(dev)
    B, D = r.shape
    w = torch.from_numpy(np.ascontiguousarray(w_lm, np.float32)).to(dev).to(dt)
    V = w.shape[0]
    w = row_tiles(w)
    g = torch.from_numpy(np.ascontiguousarray(norm_w, np.float32)).to(dev).to(dt)
    logits = torch.empty(B, V, device=dev, dtype=torch.float32)
    cv = torch.empty(1024 * B, device=dev, dtype=torch.float32)
    ci = torch.empty(1024 * B, device=dev, dtype=torch.int32)
    ticket = torch.zeros(1, device=dev, dtype=torch.int32)
    tok = torch.empty(B, device=dev, dtype=torch.int32)
    a = _native.LmArgs(dtype=dtype_bytes, batch=B, hidden=D, vocab=V, grid=0, eps=eps,
                       resid=r.data_ptr(), norm_w=g.data_ptr(), w=w.data_ptr(),
                       logits=logits.data_ptr(), cand_val=cv.data_ptr(), cand_idx=ci.data_ptr(),
                       ticket=ticket.data_ptr(), token_out=tok.data_ptr(), step_pos=None)
    _native.check(_native.lib().cfb_lm_head_argmax(a, _native.stream_ptr()))
    return logits.cpu().numpy(), tok.cpu().numpy()
