"""Generate golden vectors by running the REAL reference ``clusterdec`` package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the reference read-only from ``/root/reference/pkg/src`` and writes
``tests/golden/golden.npz`` + ``tests/golden/golden.json``.  The GPU box has no
``/root/reference``; tests there only read these committed fixtures.

Large inputs are NOT stored: the seeded generators are deterministic, so the
fixtures store a sha256 of every generated input array (pinning our own
generators bit-for-bit) plus the reference's outputs.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, REF)
    from clusterdec import collectives as coll
    from clusterdec.dataflows import (run_fused_mha_decode, run_fused_mla_decode,
                                      run_splithead_decode)
    from clusterdec.oracle import dense_mha_decode, dense_mla_decode, ffn_reference
    from clusterdec.scenarios import (ModelDims, random_mha_scenario, random_mla_scenario,
                                      with_preappended_cache)
    from clusterdec.simcore import ClusterConfig, build_cluster

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"cases": []}

    def mha_fields(sc):
        return {k: getattr(sc, k) for k in ("hidden", "w_qkv", "w_out", "k_cache", "v_cache")}

    def mla_fields(sc):
        return {k: getattr(sc, k) for k in ("hidden", "w_q", "w_up", "w_kv", "w_down", "w_out",
                                            "kv_cache")}

    def add_case(name, kind, dims, n, seed, fields, res, extra=None, store_inputs=False):
        case = {"name": name, "kind": kind, "n_blocks": n, "seed": seed,
                "dims": dict(B=dims.batch_size, D=dims.hidden_dim, n_heads=dims.n_heads,
                             H=dims.head_dim, S=dims.seq_len, rank=dims.kv_lora_rank,
                             dtype_bytes=dims.dtype_bytes),
                "input_sha": {k: sha(v) for k, v in fields.items()}}
        if res is not None:
            arrays[f"{name}/output"] = res.output
            arrays[f"{name}/score_max"] = res.score_max
            arrays[f"{name}/score_sum"] = res.score_sum
            case["stage_traffic"] = dict(res.stage_traffic)
            case["dsmem_bytes"] = res.dsmem_bytes
            case["n_events"] = len(res.ledger)
            case["global_bytes"] = res.ledger.channel_bytes("global")
        if store_inputs:
            for k, v in fields.items():
                arrays[f"{name}/in/{k}"] = v
        if extra:
            case.update(extra)
        meta["cases"].append(case)

    # ---- split_token / split_head on MHA scenarios ---------------------------
    small = [
        (1, 16, 2, 8, 5), (2, 32, 3, 16, 17), (4, 32, 1, 16, 64), (1, 32, 2, 16, 1),
        (2, 16, 1, 8, 0),
    ]
    for dtype_bytes in (4, 2):
        for i, (B, D, nh, H, S) in enumerate(small):
            dims = ModelDims(B, D, nh, H, S, dtype_bytes=dtype_bytes)
            for n in (1, 2, 4, 8):
                if H % n or D % n:
                    continue
                sc = random_mha_scenario(dims, n_blocks=n, seed=100 + i)
                dense = dense_mha_decode(sc)
                for mode in ("two_pass", "merged"):
                    res = run_fused_mha_decode(sc, stats_mode=mode)
                    name = f"st_{dtype_bytes}_{i}_n{n}_{mode}"
                    add_case(name, "split_token", dims, n, 100 + i, mha_fields(sc), res,
                             {"stats_mode": mode}, store_inputs=(mode == "two_pass"))
                    arrays[f"{name}/dense"] = dense
                res = run_splithead_decode(sc)
                add_case(f"sh_{dtype_bytes}_{i}_n{n}", "split_head", dims, n, 100 + i,
                         mha_fields(sc), res)
                if S > 0 and n > 1:
                    pre = with_preappended_cache(sc)
                    res = run_fused_mha_decode(pre, append_new_token=False)
                    add_case(f"pre_{dtype_bytes}_{i}_n{n}", "split_token_preappended",
                             pre.dims, n, 100 + i, mha_fields(pre), res,
                             {"append_new_token": False})

    # ---- fused_mla -----------------------------------------------------------
    mla_small = [(1, 16, 2, 8, 5, 8), (2, 32, 2, 16, 33, 16), (4, 32, 1, 8, 64, 16)]
    for dtype_bytes in (4, 2):
        for i, (B, D, nh, H, S, R) in enumerate(mla_small):
            dims = ModelDims(B, D, nh, H, S, kv_lora_rank=R, dtype_bytes=dtype_bytes)
            for n in (1, 2, 4, 8):
                if H % n or D % n or R % n:
                    continue
                sc = random_mla_scenario(dims, n_blocks=n, seed=200 + i)
                for mode in ("two_pass", "merged"):
                    res = run_fused_mla_decode(sc, stats_mode=mode)
                    name = f"mla_{dtype_bytes}_{i}_n{n}_{mode}"
                    add_case(name, "fused_mla", dims, n, 200 + i, mla_fields(sc), res,
                             {"stats_mode": mode}, store_inputs=(mode == "two_pass"))
                    arrays[f"{name}/dense_absorbed"] = dense_mla_decode(sc, "absorbed")
                    arrays[f"{name}/dense_original"] = dense_mla_decode(sc, "original")

    # ---- production dims (inputs regenerated from seed, pinned by sha) --------
    for n in (1, 2, 4, 8, 16):
        dims = ModelDims(1, 4096, 2, 128, 128, dtype_bytes=2)
        sc = random_mha_scenario(dims, n_blocks=n, seed=1)
        res = run_fused_mha_decode(sc)
        add_case(f"llama2h_n{n}", "split_token", dims, n, 1, mha_fields(sc), res)
        arrays[f"llama2h_n{n}/dense"] = dense_mha_decode(sc)
    dims = ModelDims(1, 4096, 32, 128, 1024, dtype_bytes=2)
    sc = random_mha_scenario(dims, n_blocks=4, seed=7)
    res = run_fused_mha_decode(sc)
    add_case("llama_full_s1k_n4", "split_token", dims, 4, 7, mha_fields(sc), res)
    arrays["llama_full_s1k_n4/dense"] = dense_mha_decode(sc)
    dims = ModelDims(1, 2048, 16, 128, 1024, kv_lora_rank=512, dtype_bytes=2)
    sc = random_mla_scenario(dims, n_blocks=4, seed=9)
    res = run_fused_mla_decode(sc)
    add_case("dsv2_full_s1k_n4", "fused_mla", dims, 4, 9, mla_fields(sc), res)
    arrays["dsv2_full_s1k_n4/dense_absorbed"] = dense_mla_decode(sc, "absorbed")

    # ---- ffn_reference ---------------------------------------------------------
    rng = np.random.default_rng(5)
    z = rng.standard_normal((2, 32)).astype(np.float32)
    w1 = (rng.standard_normal((48, 32)) * 32 ** -0.5).astype(np.float32)
    w2 = (rng.standard_normal((48, 32)) * 32 ** -0.5).astype(np.float32)
    w3 = (rng.standard_normal((32, 48)) * 48 ** -0.5).astype(np.float32)
    for k, v in dict(z=z, w1=w1, w2=w2, w3=w3).items():
        arrays[f"ffn/{k}"] = v
    for act in ("silu", "gelu", "relu", "identity"):
        arrays[f"ffn/out_{act}"] = ffn_reference(z, w1, w2, w3, act)

    # ---- collectives KATs --------------------------------------------------------
    rng = np.random.default_rng(77)
    for n in (1, 2, 4, 8, 16):
        for op in ("sum", "max", "softmax_merge"):
            size = 10
            if op == "softmax_merge":
                pays = [np.concatenate([rng.standard_normal(5) * 3, rng.uniform(0.25, 4, 5)])
                        .astype(np.float32) for _ in range(n)]
            else:
                pays = [rng.integers(-40, 40, size).astype(np.float32) for _ in range(n)]
            for dtype_bytes in (4, 2):
                cl = build_cluster(ClusterConfig(n, dtype_bytes=dtype_bytes))
                cl.alloc_all("buf", (size,))
                for blk, p in zip(cl.blocks, pays):
                    blk.store("buf", p)
                tr = coll.cluster_reduce(cl, "buf", op)
                key = f"coll/reduce_{op}_n{n}_{dtype_bytes}"
                arrays[key + "/in"] = np.stack(pays)
                arrays[key + "/out"] = np.stack([b.read("buf") for b in cl.blocks])
                meta.setdefault("collectives", {})[key] = dict(dsmem_bytes=tr.dsmem_bytes,
                                                               rounds=tr.rounds)
        seg = 3
        locs = [rng.standard_normal(seg).astype(np.float32) for _ in range(n)]
        cl = build_cluster(ClusterConfig(n))
        cl.alloc_all("g", (n * seg,))
        for blk, loc in zip(cl.blocks, locs):
            buf = np.zeros(n * seg, np.float32)
            buf[:seg] = loc
            blk.store("g", buf)
        _, tr = coll.cluster_gather(cl, "g", seg)
        key = f"coll/gather_n{n}"
        arrays[key + "/in"] = np.stack(locs)
        arrays[key + "/out"] = np.stack([b.read("g") for b in cl.blocks])
        meta.setdefault("collectives", {})[key] = dict(dsmem_bytes=tr.dsmem_bytes,
                                                       rounds=tr.rounds)

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    total = sum(v.nbytes for v in arrays.values())
    print(f"wrote {len(arrays)} arrays ({total / 1e6:.2f} MB raw), {len(meta['cases'])} cases")


if __name__ == "__main__":
    main()
