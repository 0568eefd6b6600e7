"""Benchmark: Llama2-7B batch-1 greedy decode TPOT on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--contexts 1024,2048,4096,8192,16384]

One "step" = one decode token through the whole model (embed, 32 x
[split_token attention module + fused SwiGLU FFN], LM head + argmax),
replayed from a CUDA graph with weights and KV cache resident in HBM.  The
default engine is the persistent whole-step kernel (csrc/decode_step.cu: ONE
launch per token, the attention module of each head on a 4-CTA DSMEM
cluster); the line also carries the layered engine (2 launches per layer) and
the global-memory-exchange ablation at 1K / 16K for comparison.
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
def bench_config(ctxs, world, cluster):
    """`config` of both arms (identical keys and values: the driver compares them)."""
    return {"workload": "Llama2-7B full 32-layer greedy decode, batch 1, context sweep "
                        + "/".join(str(c) for c in ctxs) + ", cluster size 4 (configs[1]); "
                        "value = mean TPOT over the sweep",
            "model": "llama2-7b", "global_batch": 1, "contexts": list(ctxs),
            "parallelism": f"tp{world}" if world > 1 else "single",
            "cluster_size": cluster,
            "l2": "inputs larger than L2 (13.5 GB weights streamed per token), no flush"}


def trace_phases(model, ctx):
    """Per-phase durations of the persistent step kernel (globaltimer stamps per
    CTA and layer): median over CTAs, mean over layers, us."""
    import torch
    tr = model.set_trace(True)
    model.set_state(ctx, 1)
    model.step()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.float64)
    model.set_trace(False)
    names = ["qkv_gemv", "attention", "o_proj", "barrier_attn", "gate_up", "barrier_ffn",
             "down_and_barrier"]
    med = np.median(np.diff(t, axis=2), axis=1).mean(axis=0) / 1e3
    layer = float(np.diff(np.median(t[:, :, 0], axis=1)).mean() / 1e3)
    return {"ctx": ctx, "layer_us": round(layer, 2),
            "phase_us": {n: round(float(v), 2) for n, v in zip(names, med)}}


def time_engine(model, ctxs, steps, warmup, cfg, world=1, replay=None):
    """CUDA-graph TPOT per context on the engine's stream (events), max over ranks."""
    import torch
    replay = replay or model.replay
    st = model.stream
    out = []
    for ctx in ctxs:
        model.set_state(ctx, 1)
        for _ in range(warmup):
            replay()
        model.set_state(ctx, 1)
        st.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        tpot_us = ms * 1e3 / steps
        mean_ctx = ctx + (steps - 1) / 2
        out.append({"ctx": ctx, "tpot_us": round(tpot_us, 2),
                    "bytes": cfg.step_bytes(int(mean_ctx)),
                    "hbm_gbs": round(cfg.step_bytes(int(mean_ctx)) / (tpot_us * 1e-6) / 1e9, 1)})
    return out


def run_ours(args, rank, world):
    import torch
    import paper_2508_18850_b200 as cfb  # noqa: F401
    from paper_2508_18850_b200 import _native
    from paper_2508_18850_b200.llama import LLAMA2_7B, LlamaDecoder
    import ctypes
    import dataclasses

    dev = torch.device("cuda", rank % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = dataclasses.replace(LLAMA2_7B, engine=args.engine)
    ctxs = [int(c) for c in args.contexts.split(",")]
    cap = max(ctxs) + args.warmup + args.steps + 8
    fused_error = None
    if world > 1 and args.tp_impl == "fused":
        # tensor parallel (configs[4]): rank-local shard, ONE persistent launch per token,
        # both all-reduces of every layer inside the kernel over NVLink peer memory.
        # Every rank must take the same path: a failure anywhere (peer mapping,
        # cross-rank wait timeout flagged by check()) sends ALL ranks to the NCCL path.
        from paper_2508_18850_b200.tp_fused import FusedTPLlama
        ok = 1
        try:
            tp = FusedTPLlama(cfg, rank, world, cap, seed=1234, nvls=args.tp_allreduce == "nvls")
            tp.set_state(ctxs[0], 1)
            tp.step()
            torch.cuda.synchronize()
            tp.check()
        except Exception as exc:  # pragma: no cover - multi-GPU only
            ok, fused_error = 0, f"{type(exc).__name__}: {str(exc)[:200]}"
        flag = torch.tensor([ok], device=dev, dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:  # pragma: no cover - multi-GPU only
            fused_error = fused_error or "another rank failed"
            args.tp_impl = "nccl"
            tp = None
            torch.cuda.empty_cache()
    if world > 1 and args.tp_impl == "fused":
        model = tp.eng
        step_fn, capture_fn, replay_fn = tp.step, tp.capture, tp.replay
        launches_per_step = tp.launches_per_step
    elif world > 1:
        # tensor parallel baseline: layered engine, one NCCL all-reduce per block half
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
    sampler = ClockSampler(dev.index or 0)
    launches = 0
    with sampler:
        sweep = time_engine(model, ctxs, args.steps, args.warmup, cfg, world, replay_fn)
        launches += launches_per_step * (args.steps + args.warmup) * len(ctxs)
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
    for s_ in sweep:
        s_["frac_of_peak"] = round(s_["hbm_gbs"] / (world * pk["hbm_gbs"]), 4)

    tpot = float(np.mean([s_["tpot_us"] for s_ in sweep]))
    e2e_tpot = float(np.mean(e2e))
    lcfg = tp.lcfg if tp is not None else cfg
    line = {
        "metric": METRIC, "value": round(tpot, 2), "unit": "us/token", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tpot / 1e3, 4),
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (random fp16 weights + KV cache, device-drawn)",
        "config": bench_config(ctxs, world, lcfg.cluster),
        "engine": (cfg.engine if world == 1 else
                   f"{tp.lcfg.engine} (fused tensor parallel: in-kernel fixed-point all-reduce over "
                   f"NVLink peer memory, 1 launch/token/rank)" if args.tp_impl == "fused" else
                   "layered (tensor parallel, NCCL between block halves)"),
        "sweep": [{k: v for k, v in s_.items() if k != "bytes"} for s_ in sweep],
        "achieved_hbm_gbs_mean": round(float(np.mean([s_["hbm_gbs"] for s_ in sweep])), 1),
        "e2e": {"value": round(e2e_tpot, 2), "unit": "us/token", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": 4,
                "path": "cfb_llama_write_token (pinned H2D) + cfb_llama_replay + cfb_llama_read "
                        "(pinned D2H) + stream sync, every step"},
    }
    traffic = None
    prof = ROOT / "profiles" / "r02" / "ncu_step_kernel_e.json"
    if world == 1 and cfg.engine == "persistent":
        # dominant kernel = the ONLY kernel of a step: llama_step_kernel<cluster>;
        # achieved = algorithmic bytes of all timed launches / their total time
        tot_b = sum(s_["bytes"] * args.steps for s_ in sweep)
        tot_t = sum(s_["tpot_us"] * 1e-6 * args.steps for s_ in sweep)
        ach = tot_b / tot_t / 1e9
        if prof.exists():
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        line["roofline"] = {
            "kernel": "llama_step_kernel<true> (whole decode step: 32 x [attention module on "
                      "4-CTA DSMEM clusters + fused SwiGLU FFN] + LM head + argmax; 1 launch/step)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "peak_kind": pk_kind,
            "unit": "GB/s", "frac": round(ach / pk["hbm_gbs"], 4), "traffic": traffic,
            "traffic_ctx": 1024 if traffic else None,
            "bytes_per_launch": {str(s_["ctx"]): s_["bytes"] for s_ in sweep},
            "avg_launch_us": {str(s_["ctx"]): s_["tpot_us"] for s_ in sweep},
            "launch_share_of_step": 1.0,
            "phases": [trace_phases(model, c) for c in (ctxs[0], ctxs[-1])]}
    line["gpu_launches"] = launches
    line["clocks"] = clocks
    if world > 1 and args.tp_impl == "fused":
        line["tp_allreduce"] = args.tp_allreduce
    if fused_error:  # pragma: no cover - multi-GPU only
        line["tp_fused_error"] = fused_error
    if world == 1 and not args.no_deepseek:
        del model
        torch.cuda.empty_cache()
        for key, fn in (("engine_compare", lambda: engine_compare(cfg, ctxs, args, pk["hbm_gbs"])),
                        ("dropin_attention_module", lambda: dropin_api(pk["hbm_gbs"])),
                        ("deepseek_block", lambda: deepseek_sweep([1024, 4096, 16384], pk["hbm_gbs"])),
                        ("deepseek_model", lambda: deepseek_model_sweep([1024, 4096, 16384], pk["hbm_gbs"])),
                        ("batch16_ffn_tcgen05", lambda: batch16_ffn(cfg, pk["hbm_gbs"])),
                        ("batch16_llama_tcgen05", lambda: batch16_stack(cfg, [1024, 4096, 16384], pk["hbm_gbs"])),
                        ("batch32_llama_tcgen05", lambda: batch16_stack(cfg, [1024, 4096], pk["hbm_gbs"], batch=32,
                                                                        kinds=("layers_only", "greedy_full")))):
            try:  # secondary configs; never lose the headline line over one of them
                line[key] = fn()
                items = line[key] if isinstance(line[key], list) else [line[key]]
                line["gpu_launches"] += sum(d.get("launches", 0) for d in items)
            except Exception as exc:
                line[key] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    if world > 1 and args.tp_impl == "fused":
        try:  # the NCCL baseline of the same TP decode (layered engine, 2L+1 collectives)
            line["tp_nccl_baseline"] = tp_nccl_baseline(cfg, rank, world, [ctxs[0], ctxs[-1]], args,
                                                        pk["hbm_gbs"])
            line["gpu_launches"] += sum(d.get("launches", 0) for d in line["tp_nccl_baseline"])
        except Exception as exc:  # pragma: no cover - multi-GPU only
            line["tp_nccl_baseline"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    if world > 1 and not args.no_deepseek:
        del model
        torch.cuda.empty_cache()
        try:  # extra configs[4] line; never lose the TPOT line over it
            # configs[4]: batch 16 at 16K context (and 1K), KV sharded by heads over the ranks
            line["batch16_tp"] = [batch16_tp(cfg, rank, world, c, pk["hbm_gbs"]) for c in (1024, 16384)]
        except Exception as exc:  # pragma: no cover - multi-GPU only
            line["batch16_tp"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        try:
            line["deepseek_tp"] = deepseek_tp(rank, world, [1024, 16384], pk["hbm_gbs"])
        except Exception as exc:  # pragma: no cover - multi-GPU only
            line["deepseek_tp"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ctxs, cfg)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return line


def dropin_api(peak_gbs, S=1024, reps=10):
    """configs[0]'s attention module through the reference-facing Python API
    (run_fused_mha_decode: host numpy scenario in, DecodeResult out): the first
    call (uploads + packs), a repeated call on the same scenario (device cache,
    checksum-validated) and calls on a prepare()d handle with a new hidden
    vector each time (weights resident)."""
    import paper_2508_18850_b200 as cfb
    dims = cfb.ModelDims(1, 4096, 32, 128, S, dtype_bytes=2)
    sc = cfb.random_mha_scenario(dims, n_blocks=4, seed=0)
    cfb.clear_device_cache()
    t0 = time.perf_counter()
    cfb.run_fused_mha_decode(sc)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(3):
        cfb.run_fused_mha_decode(sc)
    cached = (time.perf_counter() - t0) / 3
    prep = cfb.prepare(sc)
    hs = [np.random.default_rng(i).standard_normal((1, 4096)).astype(np.float16).astype(np.float32)
          for i in range(reps)]
    cfb.run_fused_mha_decode(prep.with_hidden(hs[0]))
    t0 = time.perf_counter()
    for h in hs:
        cfb.run_fused_mha_decode(prep.with_hidden(h))
    warm = (time.perf_counter() - t0) / reps
    nbytes = 150994944 + 16384 * S  # module weights + one layer of KV at S positions
    cfb.clear_device_cache()
    return {"S": S, "cluster": 4, "first_call_ms": round(cold * 1e3, 2),
            "cached_call_ms": round(cached * 1e3, 2), "prepared_call_ms": round(warm * 1e3, 3),
            "module_bytes": nbytes, "launches": 2 * (reps + 5)}


def tp_nccl_baseline(cfg, rank, world, ctxs, args, peak_gbs):
    """TP decode through the layered engine with one NCCL all-reduce per block
    half (torch.distributed, graph-captured): the baseline the fused in-kernel
    all-reduce replaces.  Max over ranks."""
    import torch
    from paper_2508_18850_b200.tp import TPLlamaDecoder
    tp = TPLlamaDecoder(cfg, rank, world, max(ctxs) + args.warmup + args.steps + 8, seed=1234)
    tp.set_state(ctxs[0], 1)
    tp.step()
    torch.cuda.synchronize()
    tp.set_state(ctxs[0], 1)
    tp.capture()
    out = []
    for s_ in time_engine(tp.eng, ctxs, args.steps, args.warmup, cfg, world, tp.replay):
        out.append({"ctx": s_["ctx"], "tpot_us": s_["tpot_us"], "hbm_gbs": s_["hbm_gbs"],
                    "frac_of_peak": round(s_["hbm_gbs"] / (world * peak_gbs), 4),
                    "launches": tp.launches_per_step * (args.steps + args.warmup)})
    del tp
    torch.cuda.empty_cache()
    return out


def engine_compare(cfg, ctxs, args, peak_gbs):
    """The other B=1 engines on the same workload: the layered engine (split_token
    cluster kernel + fused FFN kernel, 2 launches per layer), the persistent
    kernel with the cluster gather / exchange through global memory instead of
    DSMEM (same partitioning: the paper's with/without-DSMEM ablation,
    PAPER.md:889-891), the flat variant (attention split over all SMs), and the
    persistent engine on a paged KV cache (shuffled 128-position pages,
    head-major pools, `LlamaDecoder.page_kv`)."""
    import dataclasses
    import torch
    from paper_2508_18850_b200.llama import LlamaDecoder
    out = []
    for eng in ("layered", "persistent_nodsmem", "persistent_flat", "persistent_paged"):
        c = dataclasses.replace(cfg, engine=eng.replace("_paged", ""))
        m = LlamaDecoder.random(c, cache_cap=max(ctxs) + args.warmup + args.steps + 8, seed=1234)
        if eng.endswith("_paged"):
            m.page_kv(seed=1)
            torch.cuda.empty_cache()
        m.set_state(ctxs[0], 1)
        m.step()
        torch.cuda.synchronize()
        m.set_state(ctxs[0], 1)
        m.capture()
        for s_ in time_engine(m, ctxs, args.steps, args.warmup, c):
            out.append({"engine": eng, "ctx": s_["ctx"], "tpot_us": s_["tpot_us"],
                        "hbm_gbs": s_["hbm_gbs"], "frac_of_peak": round(s_["hbm_gbs"] / peak_gbs, 4),
                        "launches": m.launches_per_step * (args.steps + args.warmup)})
        del m
        torch.cuda.empty_cache()
    return out


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


def deepseek_model_sweep(ctxs, peak_gbs, steps=20):
    """configs[2] end to end: DeepSeek-V2-Lite-shaped model (27 layers of MLA
    engine + fused MoE, 102,400-token LM head + argmax), greedy TPOT from ONE
    CUDA graph per step (deepseek_model.DeepSeekDecoder; the latent caches are
    attended, not appended - reference dataflows.py:393-397)."""
    import torch
    from paper_2508_18850_b200.deepseek_model import LITE_MODEL, DeepSeekDecoder
    out = []
    for S in ctxs:
        m = DeepSeekDecoder.random(LITE_MODEL, S, seed=0)
        m.set_token(1)
        m.step()
        torch.cuda.synchronize()
        m.capture()
        for _ in range(3):
            m.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(m.stream)
        for _ in range(steps):
            m.replay()
        e1.record(m.stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / steps
        nbytes = LITE_MODEL.step_bytes(S)
        out.append({"ctx": S, "layers": LITE_MODEL.n_layers, "vocab": LITE_MODEL.vocab,
                    "tpot_us": round(us, 1), "hbm_gbs": round(nbytes / us / 1e3, 1),
                    "frac_of_peak": round(nbytes / us / 1e3 / peak_gbs, 4), "bytes": nbytes,
                    "launches": (2 + 4 * LITE_MODEL.n_layers) * (steps + 4)})
        del m
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
    m.set_positions([ctx] * m.B)
    m.reserve(4 * steps + 8)
    (m.decode_step if full else m.step)()
    torch.cuda.synchronize()
    m.set_positions([ctx] * m.B)
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


def batch16_stack(cfg, ctxs, peak_gbs, steps=10, batch=16, kinds=("layers_only", "greedy_full",
                                                                   "greedy_full_paged")):
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
        for kind in kinds:
            if kind == "greedy_full_paged":
                m = BatchedLlama.random_paged(cfg, max_len=cap, seed=0, batch=batch)
            elif kind == "layers_only" or "layers_only" not in kinds:
                m = BatchedLlama.random(cfg, cache_cap=cap, seed=0, batch=batch)
            m.random_head(cfg.vocab)
            full = kind != "layers_only"
            us = _time_b16(m, ctx, full, steps)
            gbs = m.step_bytes(ctx + 3 + steps // 2, head=full) / us / 1e3
            out.append({"ctx": ctx, "batch": batch, "step": kind,
                        "step_us": round(us, 1), "tokens_per_s": round(batch * 1e6 / us, 1),
                        "hbm_gbs": round(gbs, 1), "frac_of_peak": round(gbs / peak_gbs, 4),
                        "launches": (7 * cfg.n_layers + 1 + (4 if full else 0)) * (steps + 4)})
            if kind != "layers_only" or kind == kinds[-1]:
                del m
                torch.cuda.empty_cache()
    return out


def batch16_tp(cfg, rank, world, ctx, peak_gbs, steps=10):
    """configs[4] batch 16: 16 independent sequences, tensor-parallel shards
    (tp.TPBatchedLlama), one NCCL all-reduce of the residual per block half,
    CUDA graph per step; max over ranks."""
    import torch
    from paper_2508_18850_b200.tp import TPBatchedLlama
    torch.cuda.empty_cache()
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
def _block_weights(cfg, rng):
    """fp32 numpy weights of ONE decoder block (oracle inputs, fp16-valued)."""
    D, F, nh, H = cfg.hidden, cfg.inter, cfg.n_heads, cfg.head_dim

    def f16(shape, scale):
        return (rng.standard_normal(shape, dtype=np.float32) * scale).astype(np.float16).astype(np.float32)

    return dict(x=f16((1, D), 1.0), g1=np.ones(D, np.float32), g2=np.ones(D, np.float32),
                w_qkv=f16((nh, D, 3 * H), D ** -0.5), w_out=f16((nh, H, D), H ** -0.5),
                w1=f16((F, D), D ** -0.5), w2=f16((F, D), D ** -0.5), w3=f16((D, F), F ** -0.5))


def _kv(cfg, ctx, rng):
    def f16(shape):
        return rng.standard_normal(shape, dtype=np.float32).astype(np.float16).astype(np.float32)
    return dict(k=f16((cfg.n_heads, ctx, cfg.head_dim)), v=f16((cfg.n_heads, ctx, cfg.head_dim)))


def _block_once(cfg, w, kv):
    from oracle import clusterdec_port as cp
    from oracle import llama_port as lp
    h = lp.rmsnorm_f16(w["x"], w["g1"], cfg.eps)
    x = w["x"] + cp.dense_mha(h, w["w_qkv"], w["w_out"], kv["k"], kv["v"])
    return x + lp.ffn_block(x, w["g2"], w["w1"], w["w2"], w["w3"], cfg.eps)


def _lm_head_once(cfg, w, x):
    from oracle import llama_port as lp
    return int(np.argmax(lp.rmsnorm_f16(x, np.ones(cfg.hidden, np.float32), cfg.eps) @ w.T))


def cpu_info():
    import platform
    model = platform.processor()
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                model = l.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        blas = [f"{d['internal_api']} {d.get('version')} ({d.get('architecture')}, "
                f"{d.get('num_threads')} threads)" for d in threadpool_info() if d["user_api"] == "blas"]
    except ImportError:  # pragma: no cover
        blas = []
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "blas": blas,
            "numpy": np.__version__}


def cpu_baseline(ctxs, cfg, reps=5):
    """Oracle (numpy port of the reference path, reference oracle.py:30-52 +
    :112-131 composed into a block) timed on the host: per context one block
    (best and median of `reps` after a warm run) x 32 layers + the LM head,
    at 1 thread and at all threads."""
    from threadpoolctl import threadpool_limits
    rng = np.random.default_rng(0)
    w = _block_weights(cfg, rng)
    w_lm = (rng.standard_normal((cfg.vocab, cfg.hidden), dtype=np.float32)
            * cfg.hidden ** -0.5).astype(np.float16).astype(np.float32)
    res = {}
    for threads in (1, os.cpu_count()):
        per = {}
        with threadpool_limits(threads):
            for ctx in ctxs:
                kv = _kv(cfg, ctx, rng)
                _block_once(cfg, w, kv)  # warm
                t = []
                for _ in range(reps):
                    t0 = time.perf_counter()
                    _block_once(cfg, w, kv)
                    t.append(time.perf_counter() - t0)
                t0 = time.perf_counter()
                _lm_head_once(cfg, w_lm, w["x"])
                lm = time.perf_counter() - t0
                per[str(ctx)] = {"block_best_ms": round(min(t) * 1e3, 2),
                                 "block_median_ms": round(float(np.median(t)) * 1e3, 2),
                                 "tpot_us": round((min(t) * cfg.n_layers + lm) * 1e6, 1)}
                del kv
        res[threads] = per
    allt = res[os.cpu_count()]
    return {"value": round(float(np.mean([v["tpot_us"] for v in allt.values()])), 1),
            "unit": "us/token", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle numpy block (RMSNorm + dense_mha_decode + residual + RMSNorm + "
                      f"SwiGLU ffn_reference + residual) at each ctx {ctxs}, B=1, best of {reps} "
                      f"after a warm run, x{cfg.n_layers} layers + LM head; value = mean over "
                      f"contexts at {os.cpu_count()} threads",
            "per_ctx_all_threads": allt, "per_ctx_1_thread": res[1], "host": cpu_info()}


class contextlib_null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_reference(args, rank, world):
    """Reference arm: the oracle port of the reference's CPU path on the host
    cores, each step = one block per context x 32 layers + the LM head."""
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
    w = _block_weights(cfg, rng)
    kvs = {c: _kv(cfg, c, rng) for c in ctxs}
    w_lm = (rng.standard_normal((cfg.vocab, cfg.hidden), dtype=np.float32)
            * cfg.hidden ** -0.5).astype(np.float16).astype(np.float32)
    with lim:
        def one_step():
            per = []
            for c in ctxs:
                t0 = time.perf_counter()
                _block_once(cfg, w, kvs[c])
                blk = time.perf_counter() - t0
                t0 = time.perf_counter()
                _lm_head_once(cfg, w_lm, w["x"])
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
            "ms_per_step": round(tpot / 1e3, 3), "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32 (fp16-valued inputs)", "data": "synthetic",
            "config": bench_config(ctxs, world, _local_cluster(cfg, world, args.tp_impl)),
            "cpu_baseline": {"value": round(tpot, 1), "unit": "us/token", "cores": threads,
                             "kind": "port", "sample": sample, "host": cpu_info()},
            "e2e": {"value": round(tpot, 1), "unit": "us/token", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _local_cluster(cfg, world, tp_impl="fused"):
    """cluster size the GPU arm reports for this N (tp.local_config)."""
    if world <= 1:
        return cfg.cluster
    if tp_impl == "fused":
        from paper_2508_18850_b200.tp_fused import fused_local_config
        return fused_local_config(cfg, world).cluster
    from paper_2508_18850_b200.tp import local_config
    return local_config(cfg, world).cluster


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--contexts", default="1024,2048,4096,8192,16384")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-deepseek", action="store_true")
    ap.add_argument("--engine", default="persistent",
                    choices=["persistent", "layered", "persistent_flat", "persistent_nodsmem"])
    ap.add_argument("--tp-impl", default="fused", choices=["fused", "nccl"],
                    help="N>1: in-kernel all-reduce over peer memory (fused) or NCCL between launches")
    ap.add_argument("--tp-allreduce", default="peer", choices=["peer", "nvls"],
                    help="fused TP: sums pushed to every peer (peer) or one multimem.red on an NVLS "
                         "multicast buffer (nvls)")
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
