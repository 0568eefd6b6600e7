"""fused_mla (and split_head) dataflows on the GPU: drop-ins for the
reference's ``run_fused_mla_decode`` (``dataflows.py:316-429``) and
``run_splithead_decode`` (``dataflows.py:432-502``).

The scenario's arrays are packed once per call into the kernel layouts of
``include/cfb.h`` (``cfb_mla_args``), the kernel runs through the C ABI, and
the result carries the output, the statistics of rank 0 and the DSMEM ledger
of the kernel's static schedule, cross-checked against the byte counters the
kernel kept.  Same deliberate deviation as split_token: heads are summed in
64-bit fixed point (exact, order-free) instead of f16-rounded atomics.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .exceptions import DimensionError, SimulationError
from .fused import (FUSED_MLA, MERGED, TWO_PASS, DecodeResult, _emit_global, _finish_output,
                    padded_hidden, pow2_at_least, validate_partitioning)
from .layouts import rotated_rows, row_tiles, wo_rows
from .ledger import StageTrace, TrafficLedger, emit_gather, emit_reduce
from .scenario import validate_scenario


def _pack_mla_static(sc, cached: bool = True) -> dict:
    """MLA weights + latent cache in cfb_mla_args layouts, through the
    checksum-validated DeviceCache (or freshly built for ``prepare``)."""
    import torch
    from .devcache import CACHE
    dev = _native.require_cuda()
    d = sc.dims
    n, nb = sc.cluster.n_blocks, d.dtype_bytes
    dt = torch.float16 if nb == 2 else torch.float32
    B, D, nh, H, R = d.batch_size, d.hidden_dim, d.n_heads, d.head_dim, d.kv_lora_rank
    S = d.seq_len
    Hp, Rp = pow2_at_least(H), pow2_at_least(R)
    Dp = padded_hidden(D, n, nb)
    h, rs = H // n, R // n
    rsp = pow2_at_least(rs, 16 // nb)

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)

    def get(arr, tag, build):
        return CACHE.get(arr, ("mla",) + tag, build) if cached else build(arr)

    def b_q(a):
        wq = torch.zeros(nh, Dp, H, device=dev, dtype=dt)
        wq[:, :D, :] = up(a).to(dt)                              # (nh, Dp, H)
        return row_tiles(wq.reshape(nh, Dp, n, h).permute(0, 2, 3, 1).contiguous())  # (nh, N, h, Dp)

    def b_kv(a):
        wkv = torch.zeros(Dp, R, device=dev, dtype=dt)
        wkv[:D] = up(a).to(dt)
        return row_tiles(wkv.reshape(Dp, n, rs).permute(1, 2, 0).contiguous())       # (N, rs, Dp)

    def b_up(a):
        wup = torch.zeros(nh, Hp, R, device=dev, dtype=dt)
        wup[:, :H] = up(a).to(dt)
        return rotated_rows(wup.reshape(nh, Hp, n, rs).permute(0, 2, 3, 1).contiguous())

    def b_dn(a):
        wdn = torch.zeros(nh, n, rsp, Hp, device=dev, dtype=dt)
        wdn[:, :, :rs, :H] = up(a).to(dt).reshape(nh, n, rs, H)
        return rotated_rows(wdn.transpose(2, 3).contiguous())     # (nh, N, Hp, rsp)

    def b_out(a):
        wo = torch.zeros(nh, Dp, Hp, device=dev, dtype=dt)
        wo[:, :D, :H] = up(a).transpose(1, 2).to(dt)
        return wo_rows(wo, n)

    def b_cache(a):
        c = torch.zeros(max(S, 1), Rp, device=dev, dtype=dt)
        if S:
            c[:S, :R] = up(a).to(dt)
        return c

    key = (n, nb, Hp, Rp, Dp)
    with torch.no_grad():
        return dict(w_q=get(sc.w_q, ("q",) + key, b_q), w_kv=get(sc.w_kv, ("kv",) + key, b_kv),
                    w_up=get(sc.w_up, ("up",) + key, b_up), w_down=get(sc.w_down, ("dn",) + key, b_dn),
                    w_out=get(sc.w_out, ("out",) + key, b_out),
                    cache=get(sc.kv_cache, ("cache", S) + key, b_cache), Dp=Dp, Hp=Hp, Rp=Rp)


def pack_mla(sc, dev, dt, cached: bool = True, packed: dict | None = None):
    """DecodeScenario (MLA) -> dict of device tensors in cfb_mla_args layouts
    (static weights from the device cache / a prepared handle + the hidden)."""
    import torch
    pk = dict(packed if packed is not None else _pack_mla_static(sc, cached))
    d = sc.dims
    x = torch.zeros(d.batch_size, pk["Dp"], device=dev, dtype=dt)
    x[:, :d.hidden_dim] = torch.from_numpy(np.ascontiguousarray(sc.hidden, np.float32)).to(dev).to(dt)
    pk["x"] = x
    return pk


def run_fused_mla_decode(scenario, stats_mode: str = TWO_PASS,
                         append_new_token: bool = True) -> DecodeResult:
    """fused_mla latent attention on the GPU (one cluster per head); takes a
    scenario or its ``prepare``d handle (devcache.py)."""
    import torch
    from .devcache import PreparedScenario
    prepared = scenario if isinstance(scenario, PreparedScenario) else None
    if prepared is not None:
        scenario = prepared.scenario
    validate_partitioning(scenario, FUSED_MLA, append_new_token)
    validate_scenario(scenario)
    if stats_mode not in (TWO_PASS, MERGED):
        raise ValueError(f"unknown stats_mode {stats_mode!r}")
    dev = _native.require_cuda()
    d = scenario.dims
    n, nb = scenario.cluster.n_blocks, d.dtype_bytes
    B, D, nh, H, R = d.batch_size, d.hidden_dim, d.n_heads, d.head_dim, d.kv_lora_rank
    if B > 4:
        raise DimensionError("the fused_mla kernel supports batch <= 4")
    dt = torch.float16 if nb == 2 else torch.float32
    with torch.no_grad():
        pk = pack_mla(scenario, dev, dt, packed=prepared.packed if prepared is not None else None)
        out = torch.empty(B, pk["Dp"], device=dev, dtype=torch.float32)
        accum = torch.zeros(B, pk["Dp"], device=dev, dtype=torch.int64)
        stats = torch.zeros(nh, 2, B, device=dev, dtype=torch.float32)
        traffic = torch.zeros(16, device=dev, dtype=torch.int64)
        flags = (_native.APPEND if append_new_token else 0) | (
            _native.STATS_MERGED if stats_mode == MERGED else 0)
        args = _native.MlaArgs(
            dtype=nb, batch=B, hidden=pk["Dp"], n_heads=nh, head_dim=H, head_pad=pk["Hp"],
            kv_rank=R, rank_pad=pk["Rp"], cluster=n, seq_len=d.seq_len, flags=flags,
            x=pk["x"].data_ptr(), w_q=pk["w_q"].data_ptr(), w_kv=pk["w_kv"].data_ptr(),
            w_up=pk["w_up"].data_ptr(), w_down=pk["w_down"].data_ptr(),
            w_out=pk["w_out"].data_ptr(), cache=pk["cache"].data_ptr(), out=out.data_ptr(),
            accum=accum.data_ptr(), stats=stats.data_ptr(), traffic=traffic.data_ptr())
        _native.check(_native.lib().cfb_mla_decode(args, _native.stream_ptr()))
        torch.cuda.synchronize()
        out_np = out[:, :D].cpu().numpy()
        st = stats.cpu().numpy()
        dev_traffic = traffic.cpu().numpy()

    ledger = TrafficLedger()
    stage_traffic: dict[str, int] = {}
    traces = []
    h, rs = H // n, R // n
    for head in range(nh):
        tr = [("q_proj_gather", emit_gather(ledger, n, B * h * nb)),
              ("latent_kv_gather", emit_gather(ledger, n, B * rs * nb)),
              ("absorbed_q_gather", emit_gather(ledger, n, B * rs * nb))]
        if stats_mode == MERGED:
            tr.append(("stats_merge_reduce", emit_reduce(ledger, n, 2 * B * nb)))
        else:
            tr.append(("stats_max_reduce", emit_reduce(ledger, n, B * nb)))
            tr.append(("stats_sum_reduce", emit_reduce(ledger, n, B * nb)))
        tr.append(("attn_out_reduce", emit_reduce(ledger, n, B * R * nb)))
        tr.append(("down_proj_reduce", emit_reduce(ledger, n, B * H * nb)))
        for stage, t in tr:
            stage_traffic[stage] = stage_traffic.get(stage, 0) + t.dsmem_bytes
            traces.append(StageTrace(stage, head, t))
        _emit_global(ledger, n, B, D // n, nb)
    device_traffic = {_native.STAGE_NAMES[i]: int(dev_traffic[i]) for i in range(11)
                      if _native.STAGE_NAMES[i] in stage_traffic}
    if device_traffic != stage_traffic:
        raise SimulationError(f"kernel DSMEM byte counters {device_traffic} disagree with the "
                              f"schedule {stage_traffic}")
    return DecodeResult(output=_finish_output(out_np), ledger=ledger, stage_traffic=stage_traffic,
                        score_max=np.ascontiguousarray(st[:, 0, :]),
                        score_sum=np.ascontiguousarray(st[:, 1, :]), collectives=traces,
                        n_clusters=nh, n_blocks=n, device_traffic=device_traffic)


def run_splithead_decode(scenario, append_new_token: bool = True) -> DecodeResult:
    """split_head dataflow on the GPU (``dataflows.py:432-502``)."""
    import torch
    from .fused import SPLIT_HEAD
    validate_partitioning(scenario, SPLIT_HEAD, append_new_token)
    validate_scenario(scenario)
    dev = _native.require_cuda()
    d = scenario.dims
    n, nb = scenario.cluster.n_blocks, d.dtype_bytes
    B, D, nh, H, S = d.batch_size, d.hidden_dim, d.n_heads, d.head_dim, d.seq_len
    dt = torch.float16 if nb == 2 else torch.float32

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).to(dt)

    with torch.no_grad():
        x, wqkv, wo = up(scenario.hidden), up(scenario.w_qkv), up(scenario.w_out)
        kc = up(scenario.k_cache) if S else torch.zeros(1, device=dev, dtype=dt)
        vc = up(scenario.v_cache) if S else torch.zeros(1, device=dev, dtype=dt)
        out = torch.empty(B, D, device=dev, dtype=torch.float32)
        accum = torch.zeros(B, D, device=dev, dtype=torch.int64)
        stats = torch.zeros(nh, 2, B, device=dev, dtype=torch.float32)
        traffic = torch.zeros(16, device=dev, dtype=torch.int64)
        args = _native.SplitHeadArgs(
            dtype=nb, batch=B, hidden=D, n_heads=nh, head_dim=H, cluster=n, seq_len=S,
            flags=_native.APPEND if append_new_token else 0, x=x.data_ptr(),
            w_qkv=wqkv.data_ptr(), w_out=wo.data_ptr(), k_cache=kc.data_ptr(),
            v_cache=vc.data_ptr(), out=out.data_ptr(), accum=accum.data_ptr(),
            stats=stats.data_ptr(), traffic=traffic.data_ptr())
        _native.check(_native.lib().cfb_splithead_decode(args, _native.stream_ptr()))
        torch.cuda.synchronize()
        out_np = out.cpu().numpy()
        st = stats.cpu().numpy()
        dev_traffic = traffic.cpu().numpy()

    ledger = TrafficLedger()
    stage_traffic: dict[str, int] = {}
    traces = []
    att = S + (B if append_new_token else 0)
    for head in range(nh):
        tr = [("score_reduce", emit_reduce(ledger, n, B * att * nb)),
              ("out_proj_reduce", emit_reduce(ledger, n, B * D * nb))]
        for stage, t in tr:
            stage_traffic[stage] = stage_traffic.get(stage, 0) + t.dsmem_bytes
            traces.append(StageTrace(stage, head, t))
        for _ in range(B):  # rank 0 writes the full head output once per row
            ledger.record(-1, 0, -1, D * nb, "global")
    device_traffic = {"score_reduce": int(dev_traffic[9]), "out_proj_reduce": int(dev_traffic[10])}
    if device_traffic != stage_traffic:
        raise SimulationError(f"kernel DSMEM byte counters {device_traffic} disagree with the "
                              f"schedule {stage_traffic}")
    return DecodeResult(output=_finish_output(out_np), ledger=ledger, stage_traffic=stage_traffic,
                        score_max=np.ascontiguousarray(st[:, 0, :]),
                        score_sum=np.ascontiguousarray(st[:, 1, :]), collectives=traces,
                        n_clusters=nh, n_blocks=n, device_traffic=device_traffic)
