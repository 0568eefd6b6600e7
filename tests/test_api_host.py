"""Host-side (CPU) tests of the drop-in API: generators, validation, ledger
model, and the C-ABI library's exported symbols.  No GPU needed."""

from __future__ import annotations

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2508_18850_b200 as cfb
from paper_2508_18850_b200 import _native
from paper_2508_18850_b200.ledger import TrafficLedger, emit_gather, emit_reduce

ROOT = Path(__file__).resolve().parents[1]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def test_product_generators_reproduce_reference_draws(golden):
    meta, _ = golden
    checked = 0
    for case in meta["cases"]:
        d = case["dims"]
        if case["kind"] == "split_token_preappended":
            continue
        dims = cfb.ModelDims(d["B"], d["D"], d["n_heads"], d["H"], d["S"], d["rank"],
                             d["dtype_bytes"])
        if case["kind"] == "fused_mla":
            sc = cfb.random_mla_scenario(dims, n_blocks=case["n_blocks"], seed=case["seed"])
        else:
            sc = cfb.random_mha_scenario(dims, n_blocks=case["n_blocks"], seed=case["seed"])
        for k, h in case["input_sha"].items():
            assert _sha(getattr(sc, k)) == h, (case["name"], k)
        checked += 1
    assert checked > 50


def test_preappended_cache_matches_reference_inputs(golden):
    meta, _ = golden
    for case in meta["cases"]:
        if case["kind"] != "split_token_preappended":
            continue
        d = case["dims"]
        dims = cfb.ModelDims(d["B"], d["D"], d["n_heads"], d["H"], d["S"] - d["B"],
                             dtype_bytes=d["dtype_bytes"])
        pre = cfb.with_preappended_cache(cfb.random_mha_scenario(dims, case["n_blocks"],
                                                                 case["seed"]))
        for k, h in case["input_sha"].items():
            assert _sha(getattr(pre, k)) == h, (case["name"], k)


def test_validation_errors_match_reference_types():
    with pytest.raises(cfb.InvalidClusterSize):
        cfb.ClusterConfig(3)
    with pytest.raises(cfb.DimensionError):
        cfb.ModelDims(0, 8, 1, 4, 2)
    dims = cfb.ModelDims(1, 8, 1, 6, 2)
    sc = cfb.random_mha_scenario(dims, n_blocks=4, seed=0)
    with pytest.raises(cfb.DimensionError):
        cfb.validate_partitioning(sc, "split_token")
    with pytest.raises(cfb.DimensionError):
        cfb.validate_partitioning(sc, "pipelined")
    with pytest.raises(cfb.DimensionError):
        cfb.run_dataflow("pipelined", sc)
    bare = cfb.random_mha_scenario(cfb.ModelDims(1, 8, 1, 4, 0), n_blocks=2, seed=0)
    with pytest.raises(cfb.DimensionError):
        cfb.validate_partitioning(bare, "split_token", append_new_token=False)
    mla = cfb.random_mla_scenario(cfb.ModelDims(1, 8, 1, 8, 2, kv_lora_rank=6), n_blocks=4)
    with pytest.raises(cfb.DimensionError):
        cfb.validate_partitioning(mla, "fused_mla")
    with pytest.raises(cfb.DimensionError):
        cfb.validate_partitioning(sc, "fused_mla")
    sc.w_out = sc.w_out[:, :, :4]
    with pytest.raises(cfb.ShapeMismatch):
        sc.validate()


def test_sequence_segments_kats():
    assert cfb.sequence_segments(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert cfb.sequence_segments(5, 4) == [(0, 2), (2, 4), (4, 5), (5, 5)]
    assert cfb.sequence_segments(0, 2) == [(0, 0), (0, 0)]
    assert cfb.sequence_segments(7, 1) == [(0, 7)]


def test_traffic_formula_kats():
    assert cfb.traffic_reduce(1024, 4) == 8192
    assert cfb.traffic_reduce(256 * 1024, 4) == 2097152
    assert cfb.traffic_gather(1024, 4) == 12288
    assert cfb.traffic_gather(1024, 16) == 245760
    for n in (1, 2, 4, 8, 16):
        led = TrafficLedger()
        assert emit_reduce(led, n, 100).dsmem_bytes == cfb.traffic_reduce(100, n)
        assert led.channel_bytes() == cfb.traffic_reduce(100, n)
        led = TrafficLedger()
        tr = emit_gather(led, n, 64)
        assert tr.dsmem_bytes == cfb.traffic_gather(64, n) == led.channel_bytes()
        per_block0 = sum(e.nbytes for e in led.events if e.src_rank == 0)
        assert per_block0 == 64 * (n - 1)


@pytest.mark.parametrize("n,expect", [(2, 1280 + 8), (4, 4352 + 32), (8, 11520 + 96),
                                      (16, 27904 + 256)])
def test_llama_split_token_budget(n, expect):
    """SURVEY §8(a) last row: Llama B=1 f16 per-cluster DSMEM bytes."""
    dims = cfb.ModelDims(1, 4096, 32, 128, 1024, dtype_bytes=2)
    bd = cfb.dataflow_traffic("split_token", dims, n)
    assert bd.headline_bytes + bd.stats_bytes == expect


def test_dataflow_traffic_matches_reference_stage_tallies(golden):
    meta, _ = golden
    for case in meta["cases"]:
        if "stage_traffic" not in case or case["kind"] == "split_token_preappended":
            continue
        d = case["dims"]
        dims = cfb.ModelDims(d["B"], d["D"], d["n_heads"], d["H"], d["S"], d["rank"],
                             d["dtype_bytes"])
        bd = cfb.dataflow_traffic(case["kind"], dims, case["n_blocks"],
                                  case.get("stats_mode", "two_pass"))
        for e in bd.entries:
            assert case["stage_traffic"][e.stage] == e.analytical_bytes * d["n_heads"]


def _declared_symbols():
    text = (ROOT / "include" / "cfb.h").read_text()
    return sorted(set(re.findall(r"\b(cfb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    syms = _declared_symbols()
    assert "cfb_mha_decode" in syms
    for s in syms:
        assert hasattr(L, s), s
    assert L.cfb_version().startswith(b"cfb")


def _struct_fields(text, name):
    body = text.split(f"typedef struct {name} {{")[1].split(f"}} {name};")[0]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        # "int batch, hidden" -> several names; drop the type words
        words = decl.replace("*", " ").replace(",", " , ").split()
        while words and words[0] in ("const", "unsigned", "long", "int", "float", "void", "char"):
            words.pop(0)
        for nm in " ".join(words).split(","):
            names.append(nm.strip().split()[-1])
    return names


@pytest.mark.parametrize("cname,pyname", [("cfb_mha_args", "MhaArgs"), ("cfb_ffn_args", "FfnArgs"),
                                          ("cfb_lm_args", "LmArgs"), ("cfb_mla_args", "MlaArgs"),
                                          ("cfb_splithead_args", "SplitHeadArgs"),
                                          ("cfb_moe_args", "MoeArgs"),
                                          ("cfb_mla_engine_args", "MlaEngineArgs"),
                                          ("cfb_ffn_b16_args", "FfnB16Args"),
                                          ("cfb_b16_layer_args", "B16LayerArgs")])
def test_abi_struct_layout_matches_header(cname, pyname):
    """ctypes mirrors must have the field order of the C structs."""
    text = (ROOT / "include" / "cfb.h").read_text()
    assert _struct_fields(text, cname) == [f[0] for f in getattr(_native, pyname)._fields_]


def test_wo_rows_layout():
    """W_out^T rank slices with per-row chunk rotation (logical chunk k of slice
    row g at physical chunk (k + g) mod nch)."""
    import torch
    from paper_2508_18850_b200.layouts import wo_rows
    nh, D, Hp, N = 2, 24, 32, 4  # cols = 6, nch = 4 (fp16)
    w = torch.arange(nh * D * Hp, dtype=torch.float32).reshape(nh, D, Hp).half()
    t = wo_rows(w, N)
    assert t.shape == (nh, N, 6, Hp)
    for h in range(nh):
        for r in range(N):
            for g in range(6):
                for k in range(4):
                    p = (k + g) % 4
                    assert torch.equal(t[h, r, g, p * 8:(p + 1) * 8], w[h, r * 6 + g, k * 8:(k + 1) * 8])


def test_moe_down_blocks_layout():
    """W_down (D, F) -> [F/8][Q][8][D/Q]: block (g, q) row r = W_down^T row
    8g + r, columns q*D/Q .. (q+1)*D/Q."""
    import torch
    from paper_2508_18850_b200.moe import down_blocks, moe_segments
    for D, F in ((64, 16), (1024, 24), (2048, 16)):
        Q = moe_segments(D)
        w = torch.arange(D * F, dtype=torch.float32).reshape(D, F)
        t = down_blocks(w)
        assert t.shape == (F // 8, Q, 8, D // Q)
        for g in range(F // 8):
            for q in range(Q):
                for r in range(8):
                    assert torch.equal(t[g, q, r], w[q * D // Q:(q + 1) * D // Q, 8 * g + r])
