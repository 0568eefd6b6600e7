"""Benchmark: Llama2-7B batch-1 greedy decode TPOT on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--contexts 1024,2048,4096,8192,16384]

One "step" = one decode token through the whole model (embed, 32 x
[split_token attention module + fused SwiGLU FFN], LM head + argmax),
replayed from a CUDA graph with weights and KV cache resident in HBM.
`value` is the mean TPOT (µs/token) over the context sweep; the per-context
numbers are in `sweep`.  Inputs (13.5 GB of weights) are far larger than the
126 MB L2, so no L2 flush is needed between steps.

Under torchrun (N > 1) each rank holds a tensor-parallel shard (configs[4]:
heads, FFN columns and LM-head rows split N ways) and a step carries one NCCL
all-reduce per block half; `value` is then the TP TPOT ("scaling": "strong").
At N = 1 the line also carries `deepseek_block` (configs[2]: MLA + MoE block
latency over contexts, CUDA-graph replay of 4 distinct blocks).

--impl reference times the CPU oracle restatement of the reference path
(oracle/, numpy, all host threads) on a bounded sample: one decoder block per
context, extrapolated to 32 layers plus the LM head.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TPOT µs/token, Llama2-7B bs1 decode 1K–16K ctx; achieved HBM GB/s vs peak"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world):
    import torch
    import paper_2508_18850_b200 as cfb  # noqa: F401
    from paper_2508_18850_b200 import _native
    from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder
    import ctypes

    dev = torch.device("cuda", rank % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = LLAMA2_7B
    ctxs = [int(c) for c in args.contexts.split(",")]
    cap = max(ctxs) + args.warmup + args.steps + 8
    if world > 1:
        # tensor parallel (configs[4]): rank-local shard, one NCCL all-reduce per block half
        from paper_2508_18850_b200.tp import TPLlamaDecoder
        tp = TPLlamaDecoder(cfg, rank, world, cap, seed=1234 + rank)
        model = tp.eng
        step_fn, capture_fn, replay_fn = tp.step, tp.capture, tp.replay
        launches_per_step = tp.launches_per_step
    else:
        tp = None
        model = LlamaDecoder.random(cfg, cache_cap=cap, seed=1234 + rank)
        step_fn, capture_fn, replay_fn = model.step, model.capture, model.replay
        launches_per_step = model.launches_per_step
    L = _native.lib()
    st = model.stream

    # configure kernels outside capture, then capture one step
    model.set_state(ctxs[0], 1)
    step_fn()
    torch.cuda.synchronize()
    model.set_state(ctxs[0], 1)
    capture_fn()
    pk, pk_kind = peaks()
    sweep = []
    sampler = ClockSampler(dev.index or 0)
    launches = 0
    with sampler:
        for ctx in ctxs:
            model.set_state(ctx, 1)
            for _ in range(args.warmup):
                replay_fn()
            model.set_state(ctx, 1)
            st.synchronize()
            if world > 1:
                torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.steps):
                replay_fn()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ms], device=dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms = float(t.item())
            launches += launches_per_step * args.steps
            tpot_us = ms * 1e3 / args.steps
            mean_ctx = ctx + (args.steps - 1) / 2
            gbs = cfg.step_bytes(int(mean_ctx)) / (tpot_us * 1e-6) / 1e9  # whole job, all ranks
            sweep.append({"ctx": ctx, "tpot_us": round(tpot_us, 2), "hbm_gbs": round(gbs, 1),
                          "frac_of_peak": round(gbs / (world * pk["hbm_gbs"]), 4)})

        # e2e: host token -> device (pinned H2D), graph, token -> host (pinned D2H), per step
        host_in = torch.ones(1, dtype=torch.int32).pin_memory()
        host_out = torch.zeros(1, dtype=torch.int32).pin_memory()
        e2e = []
        for ctx in ctxs:
            model.set_state(ctx, 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                _native.check(L.cfb_llama_write_token(model._h, ctypes.c_void_p(host_in.data_ptr()),
                                                      model._sp()))
                replay_fn()
                _native.check(L.cfb_llama_read(model._h, ctypes.c_void_p(host_out.data_ptr()),
                                               None, model._sp()))
                st.synchronize()
                host_in[0] = host_out[0]
            dt = time.perf_counter() - t0
            e2e.append(dt * 1e6 / args.steps)
            launches += launches_per_step * args.steps
    clocks = sampler.summary()

    # dominant kernel (fused FFN, 64% of weight bytes): avg launch duration with
    # CUDA events on its stream, cycling through the 32 layers' weights
    lcfg = tp.lcfg if tp is not None else cfg
    ffn_bytes = 3 * lcfg.hidden * lcfg.inter * 2 + lcfg.hidden * 2
    resid = torch.randn(1, cfg.hidden, device=dev)
    out = torch.empty(1, cfg.hidden, device=dev)
    act = torch.empty(lcfg.inter, device=dev, dtype=torch.float16)
    bar = torch.zeros(1, device=dev, dtype=torch.int64)
    accum = torch.zeros(1, cfg.hidden, device=dev, dtype=torch.int64)
    fargs = []
    for lyr in model.layers:
        fargs.append(_native.FfnArgs(
            dtype=2, batch=1, hidden=cfg.hidden, inter=lcfg.inter,
            flags=_native.NORM | _native.RESID | _native.PDL, grid=0, eps=cfg.eps, x=None,
            resid=resid.data_ptr(), accum=accum.data_ptr(), norm_w=lyr["ffn_norm"].data_ptr(), w_gu=lyr["w_gu"].data_ptr(),
            w_dn=lyr["w_dn"].data_ptr(), act=act.data_ptr(), out=out.data_ptr(),
            barrier=bar.data_ptr()))
    torch.cuda.synchronize()
    for a in fargs[:4]:
        _native.check(L.cfb_ffn_decode(a, model._sp()))
    reps = 4 * len(fargs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(reps):
        _native.check(L.cfb_ffn_decode(fargs[i % len(fargs)], model._sp()))
    e1.record(st)
    torch.cuda.synchronize()
    ffn_us = e0.elapsed_time(e1) * 1e3 / reps
    launches += reps
    ffn_gbs = ffn_bytes / (ffn_us * 1e-6) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ffn_dram_bytes.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")

    tpot = float(np.mean([s["tpot_us"] for s in sweep]))
    e2e_tpot = float(np.mean(e2e))
    line = {
        "metric": METRIC, "value": round(tpot, 2), "unit": "us/token", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tpot / 1e3, 4),
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic (random fp16 weights + KV cache, device-drawn)",
        "config": {"workload": "Llama2-7B full 32-layer greedy decode, batch 1, context sweep "
                               + "/".join(str(c) for c in ctxs) + ", cluster size 4 (configs[1]); "
                               "value = mean TPOT over the sweep",
                   "model": "llama2-7b", "global_batch": 1, "contexts": ctxs,
                   "parallelism": f"tp{world}" if world > 1 else "single",
                   "cluster_size": lcfg.cluster,
                   "l2": "inputs larger than L2 (13.5 GB weights streamed per token), no flush"},
        "sweep": sweep,
        "achieved_hbm_gbs_mean": round(float(np.mean([s["hbm_gbs"] for s in sweep])), 1),
        "e2e": {"value": round(e2e_tpot, 2), "unit": "us/token", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": 4,
                "path": "cfb_llama_write_token (pinned H2D) + cfb_llama_replay + cfb_llama_read "
                        "(pinned D2H) + stream sync, every step"},
        "roofline": {"kernel": "ffn_swiglu_kernel (fused gate/up + SiLU*mul + down)",
                     "bound": "hbm", "achieved": round(ffn_gbs, 1), "peak": pk["hbm_gbs"],
                     "peak_kind": pk_kind, "unit": "GB/s", "frac": round(ffn_gbs / pk["hbm_gbs"], 4),
                     "traffic": traffic, "bytes_per_launch": ffn_bytes,
                     "avg_launch_us": round(ffn_us, 2)},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if world == 1 and not args.no_deepseek:
        del model, fargs
        torch.cuda.empty_cache()
        for key, fn in (("deepseek_block", lambda: deepseek_sweep([1024, 4096, 16384], pk["hbm_gbs"])),
                        ("batch16_ffn_tcgen05", lambda: batch16_ffn(cfg, pk["hbm_gbs"])),
                        ("batch16_llama_tcgen05", lambda: batch16_stack(cfg, [1024, 4096], pk["hbm_gbs"]))):
            try:  # secondary configs; never lose the headline line over one of them
                line[key] = fn()
                items = line[key] if isinstance(line[key], list) else [line[key]]
                line["gpu_launches"] += sum(d.get("launches", 0) for d in items)
            except Exception as exc:
                line[key] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    if world > 1 and not args.no_deepseek:
        del model, fargs
        torch.cuda.empty_cache()
        try:  # extra configs[4] line; never lose the TPOT line over it
            line["batch16_tp"] = batch16_tp(cfg, rank, world, 1024, pk["hbm_gbs"])
        except Exception as exc:  # pragma: no cover - multi-GPU only
            line["batch16_tp"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        try:
            line["deepseek_tp"] = deepseek_tp(rank, world, [1024, 16384], pk["hbm_gbs"])
        except Exception as exc:  # pragma: no cover - multi-GPU only
            line["deepseek_tp"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ctxs[:1], cfg, threads=os.cpu_count(), reps=1)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return line


def deepseek_sweep(ctxs, peak_gbs, layers=4, reps=16):
    """configs[2]: DeepSeek-V2-Lite-shaped block (fused_mla + fused MoE, PDL),
    CUDA graph of `layers` distinct blocks (nothing reused from L2)."""
    import torch
    from paper_2508_18850_b200.deepseek import LITE, DeepSeekBlock
    out = []
    for S in ctxs:
        blocks = [DeepSeekBlock.random(LITE, S, seed=s) for s in range(layers)]
        st = torch.cuda.Stream()
        resid = torch.randn(1, LITE.hidden, device="cuda")
        with torch.cuda.stream(st):
            for b in blocks:
                b.launch(resid, stream=st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for b in blocks:
                b.launch(resid, stream=st)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
        gbs = LITE.block_bytes(S) / us / 1e3
        out.append({"ctx": S, "block_us": round(us, 2), "hbm_gbs": round(gbs, 1),
                    "frac_of_peak": round(gbs / peak_gbs, 4), "bytes": LITE.block_bytes(S),
                    "launches": 2 * layers * (reps + 4)})
        del blocks, g
        torch.cuda.empty_cache()
    return out


def batch16_ffn(cfg, peak_gbs, sets=3, reps=30):
    """Batch-16 Llama2-7B FFN block on tcgen05 (tc.TcFfnB16: RMSNorm -> [w1;w2]
    projection with SwiGLU epilogue -> w3 projection with residual epilogue)."""
    import torch
    from paper_2508_18850_b200.tc import TcFfnB16
    D, F = cfg.hidden, cfg.inter
    ffns = [TcFfnB16(torch.randn(F, D, device="cuda") * D ** -0.5,
                     torch.randn(F, D, device="cuda") * D ** -0.5,
                     torch.randn(D, F, device="cuda") * F ** -0.5, torch.ones(D, device="cuda"))
            for _ in range(sets)]
    resid = torch.randn(16, D, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for f in ffns:
            f.launch(resid, pdl=True, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for r in range(reps):
            ffns[r % sets].launch(resid, pdl=True, stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    gbs = ffns[0].weight_bytes / us / 1e3
    out = {"batch": 16, "us_per_block": round(us, 2), "hbm_gbs": round(gbs, 1),
           "frac_of_peak": round(gbs / peak_gbs, 4), "tokens_per_s": round(16e6 / us, 1),
           "launches": 3 * (reps + sets)}
    del ffns
    torch.cuda.empty_cache()
    return out


def _time_b16(m, ctx, full, steps):
    import torch
    m.set_positions([ctx] * 16)
    m.reserve(4 * steps + 8)
    (m.decode_step if full else m.step)()
    torch.cuda.synchronize()
    m.set_positions([ctx] * 16)
    (m.capture_decode if full else m.capture)()
    for _ in range(3):
        m.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    for _ in range(steps):
        m.replay()
    e1.record(m.stream)
    torch.cuda.synchronize()
    m.graph = None
    return e0.elapsed_time(e1) * 1e3 / steps


def batch16_stack(cfg, ctxs, peak_gbs, steps=10):
    """Batch 16 independent sequences through the 32-layer Llama2-7B stack
    (batched.BatchedLlama: tcgen05 projections, per-sequence KV caches), CUDA
    graph per step.  Lines per context: the layer stack alone, the full greedy
    step (embed -> 32 layers -> final norm + tcgen05 LM head -> argmax -> next
    tokens), and the full step over the paged KV cache (shuffled 128-position
    pages, block table)."""
    import torch
    from paper_2508_18850_b200.batched import BatchedLlama
    out = []
    for ctx in ctxs:
        cap = ctx + 6 * steps + 16
        for kind in ("layers_only", "greedy_full", "greedy_full_paged"):
            if kind == "greedy_full_paged":
                m = BatchedLlama.random_paged(cfg, max_len=cap, seed=0)
            elif kind == "layers_only":
                m = BatchedLlama.random(cfg, cache_cap=cap, seed=0)
            m.random_head(cfg.vocab)
            full = kind != "layers_only"
            us = _time_b16(m, ctx, full, steps)
            gbs = m.step_bytes(ctx + 3 + steps // 2, head=full) / us / 1e3
            out.append({"ctx": ctx, "batch": 16, "step": kind,
                        "step_us": round(us, 1), "tokens_per_s": round(16e6 / us, 1),
                        "hbm_gbs": round(gbs, 1), "frac_of_peak": round(gbs / peak_gbs, 4),
                        "launches": (7 * cfg.n_layers + 1 + (4 if full else 0)) * (steps + 4)})
            if kind != "layers_only":
                del m
                torch.cuda.empty_cache()
    return out


def batch16_tp(cfg, rank, world, ctx, peak_gbs, steps=10):
    """configs[4] batch 16: 16 independent sequences, tensor-parallel shards
    (tp.TPBatchedLlama), one NCCL all-reduce of the residual per block half,
    CUDA graph per step; max over ranks."""
    import torch
    from paper_2508_18850_b200.tp import TPBatchedLlama
    m = TPBatchedLlama(cfg, rank, world, ctx + 3 * steps + 8, seed=rank)
    m.m.set_positions([ctx] * 16)
    m.step()
    torch.cuda.synchronize()
    m.m.set_positions([ctx] * 16)
    m.capture()
    for _ in range(3):
        m.replay()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.m.stream)
    for _ in range(steps):
        m.replay()
    e1.record(m.m.stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / steps], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    us = float(t.item())
    from paper_2508_18850_b200.batched import BatchedLlama  # noqa: F401
    nbytes = m.m.step_bytes(ctx + 3 + steps // 2) * world  # per-rank bytes x ranks (weights/KV sharded)
    return {"ctx": ctx, "batch": 16, "tp": world, "step_us": round(us, 1),
            "tokens_per_s": round(16e6 / us, 1), "hbm_gbs_all_ranks": round(nbytes / us / 1e3, 1)}


def deepseek_tp(rank, world, ctxs, peak_gbs, layers=4, reps=16):
    """DeepSeek-V2-Lite block, tensor parallel (tp.TPDeepSeekBlock): MLA
    heads and expert rows sharded, one int64 and one fp32 NCCL all-reduce per
    block; ``layers`` distinct blocks per CUDA graph; max over ranks."""
    import torch
    from paper_2508_18850_b200.deepseek import LITE
    from paper_2508_18850_b200.tp import TPDeepSeekBlock, deepseek_local_dims
    red = TPDeepSeekBlock.nccl_reducers() if world > 1 else (None, None)
    ld = deepseek_local_dims(LITE, world)
    out = []
    for ctx in ctxs:
        blocks = [TPDeepSeekBlock.random(LITE, rank, world, ctx, seed=l, reduce_int=red[0], reduce_f32=red[1])
                  for l in range(layers)]
        resid = torch.full((1, LITE.hidden), 0.5, device="cuda")
        st = torch.cuda.Stream()
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for b in blocks:
                b.launch(resid)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for b in blocks:
                b.launch(resid)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(reps):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e3 / (reps * layers)], device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        us = float(t.item())
        nbytes = ld.block_bytes(ctx) * world
        out.append({"ctx": ctx, "tp": world, "block_us": round(us, 2),
                    "hbm_gbs_all_ranks": round(nbytes / us / 1e3, 1),
                    "launches": (3 + 1) * layers * (reps + 3)})
        del g, blocks
        torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------- CPU arm
def _block_sample(cfg, ctx, rng):
    """fp32 numpy weights of ONE decoder block + a ctx-long cache (oracle inputs)."""
    from oracle import clusterdec_port as cp  # noqa: F401
    D, F, nh, H = cfg.hidden, cfg.inter, cfg.n_heads, cfg.head_dim

    def f16(shape, scale):
        return (rng.standard_normal(shape, dtype=np.float32) * scale).astype(np.float16).astype(np.float32)

    return dict(x=f16((1, D), 1.0), g1=np.ones(D, np.float32), g2=np.ones(D, np.float32),
                w_qkv=f16((nh, D, 3 * H), D ** -0.5), w_out=f16((nh, H, D), H ** -0.5),
                w1=f16((F, D), D ** -0.5), w2=f16((F, D), D ** -0.5), w3=f16((D, F), F ** -0.5),
                k=f16((nh, ctx, H), 1.0), v=f16((nh, ctx, H), 1.0))


def _block_once(cfg, s):
    from oracle import clusterdec_port as cp
    from oracle import llama_port as lp
    h = lp.rmsnorm_f16(s["x"], s["g1"], cfg.eps)
    x = s["x"] + cp.dense_mha(h, s["w_qkv"], s["w_out"], s["k"], s["v"])
    return x + lp.ffn_block(x, s["g2"], s["w1"], s["w2"], s["w3"], cfg.eps)


def _lm_head_once(cfg, w, x):
    from oracle import llama_port as lp
    return int(np.argmax(lp.rmsnorm_f16(x, np.ones(cfg.hidden, np.float32), cfg.eps) @ w.T))


def cpu_baseline(ctxs, cfg, threads, reps=1):
    """Oracle (numpy port of the reference path) timed on the host: one block
    per context x 32 layers + the LM head = TPOT estimate."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    rng = np.random.default_rng(0)
    w_lm = (rng.standard_normal((cfg.vocab, cfg.hidden), dtype=np.float32)
            * cfg.hidden ** -0.5).astype(np.float16).astype(np.float32)
    vals = []
    ctx_ = contextlib_null() if threadpool_limits is None else threadpool_limits(threads)
    with ctx_:
        for ctx in ctxs:
            s = _block_sample(cfg, ctx, rng)
            _block_once(cfg, s)  # warm
            t = []
            for _ in range(reps):
                t0 = time.perf_counter()
                _block_once(cfg, s)
                t.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            _lm_head_once(cfg, w_lm, s["x"])
            lm = time.perf_counter() - t0
            vals.append((min(t) * cfg.n_layers + lm) * 1e6)
            del s
    return {"value": round(float(np.mean(vals)), 1), "unit": "us/token", "cores": threads,
            "kind": "port",
            "sample": f"oracle numpy block (RMSNorm + dense_mha_decode + residual + RMSNorm + "
                      f"SwiGLU ffn_reference + residual) at ctx {','.join(map(str, ctxs))}, B=1, "
                      f"best of {reps}, x{cfg.n_layers} layers + LM head; OpenBLAS, {threads} threads"}


class contextlib_null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_reference(args, rank, world):
    from paper_2508_18850_b200.llama import LLAMA2_7B
    cfg = LLAMA2_7B
    ctxs = [int(c) for c in args.contexts.split(",")]
    threads = os.cpu_count()
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(threads)
    except ImportError:
        lim = contextlib_null()
    rng = np.random.default_rng(0)
    samples = {c: _block_sample(cfg, c, rng) for c in ctxs}
    w_lm = (rng.standard_normal((cfg.vocab, cfg.hidden), dtype=np.float32)
            * cfg.hidden ** -0.5).astype(np.float16).astype(np.float32)
    with lim:
        def one_step():
            per = []
            for c in ctxs:
                t0 = time.perf_counter()
                _block_once(cfg, samples[c])
                blk = time.perf_counter() - t0
                t0 = time.perf_counter()
                _lm_head_once(cfg, w_lm, samples[c]["x"])
                per.append((blk * cfg.n_layers + (time.perf_counter() - t0)) * 1e6)
            return float(np.mean(per))
        for _ in range(args.warmup):
            one_step()
        vals = [one_step() for _ in range(args.steps)]
    tpot = float(np.mean(vals))
    sample = (f"per step: one oracle decoder block (numpy port of dense_mha_decode + "
              f"ffn_reference silu + RMSNorm/residual) at each ctx {ctxs}, x{cfg.n_layers} layers "
              f"+ LM head, mean over contexts; {threads} threads")
    return {"metric": METRIC, "impl": "reference", "value": round(tpot, 1), "unit": "us/token",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tpot / 1e3, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (fp16-valued inputs)", "data": "synthetic",
            "config": {"workload": "Llama2-7B full 32-layer greedy decode, batch 1, context sweep "
                                   + "/".join(map(str, ctxs)) + " (configs[1]); value = mean TPOT",
                       "model": "llama2-7b", "global_batch": 1, "contexts": ctxs,
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": round(tpot, 1), "unit": "us/token", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(tpot, 1), "unit": "us/token", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--contexts", default="1024,2048,4096,8192,16384")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-deepseek", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.gpus else 1))
    if "RANK" not in os.environ:
        world = 1
    if args.impl == "reference":
        if rank != 0:
            return
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
