"""Golden vectors for the DeepSeek-V2 MoE layer, produced by ``transformers``'
own ``DeepseekV2Moe`` module (the reference has no MoE: SPEC.md:12, :366).

Run in the build container:

    python tests/golden/make_moe_golden.py

For every case it builds the MoE weights with ``oracle.deepseek_port.gen_moe``
(seeded, deterministic), loads them into ``DeepseekV2Moe`` (fp32, CPU, eager
expert loop), runs the layer on seeded fp16-valued token rows and stores the
output, the routed expert ids (as a sorted set per row) and a sha256 of every
weight/input array so the generator itself is pinned.  Writes
``tests/golden/moe_golden.npz`` + ``moe_golden.json``.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

CASES = [
    # name, D, E, K, F, n_shared, B, seed, scale
    ("tiny_b1", 64, 8, 2, 16, 2, 1, 0, 1.0),
    ("tiny_b3", 64, 8, 2, 16, 2, 3, 1, 1.0),
    ("tiny_noshared", 64, 8, 3, 16, 0, 2, 2, 1.0),
    ("small_b1", 256, 16, 4, 64, 1, 1, 3, 1.0),
    ("small_b4", 256, 16, 4, 64, 2, 4, 4, 2.5),
    ("mid_b2", 512, 32, 6, 128, 2, 2, 5, 1.0),
    ("lite_b1", 2048, 64, 6, 1408, 2, 1, 6, 1.0),
    ("lite_b1_s7", 2048, 64, 6, 1408, 2, 1, 7, 1.0),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def hidden_rows(B, D, seed):
    from oracle.llama_port import f16
    return f16(np.random.default_rng(seed + 12345).standard_normal((B, D), dtype=np.float32))


def weights_sha(w) -> str:
    h = hashlib.sha256()
    for a in [w["router"]] + [x for e in w["experts"] for x in (e["gate"], e["up"], e["down"])] + (
            [w["shared"][k] for k in ("gate", "up", "down")] if w["shared"] else []):
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


def main() -> None:
    import torch
    from transformers.models.deepseek_v2.configuration_deepseek_v2 import DeepseekV2Config
    from transformers.models.deepseek_v2.modeling_deepseek_v2 import DeepseekV2Moe

    from oracle import deepseek_port as dp

    torch.set_num_threads(8)
    arrays, meta = {}, {"generator": "transformers.models.deepseek_v2.DeepseekV2Moe",
                        "transformers_version": __import__("transformers").__version__,
                        "cases": []}
    for name, D, E, K, F, ns, B, seed, scale in CASES:
        w = dp.gen_moe(D, E, F, ns, seed)
        cfg = DeepseekV2Config(hidden_size=D, n_routed_experts=E, num_experts_per_tok=K,
                               moe_intermediate_size=F, n_shared_experts=ns,
                               hidden_act="silu", topk_method="greedy",
                               routed_scaling_factor=scale, norm_topk_prob=False)
        m = DeepseekV2Moe(cfg).eval()
        with torch.no_grad():
            m.gate.weight.copy_(torch.from_numpy(w["router"]))
            m.experts.gate_up_proj.copy_(torch.from_numpy(np.stack(
                [np.concatenate([e["gate"], e["up"]], 0) for e in w["experts"]])))
            m.experts.down_proj.copy_(torch.from_numpy(np.stack([e["down"] for e in w["experts"]])))
            if ns:
                m.shared_experts.gate_proj.weight.copy_(torch.from_numpy(w["shared"]["gate"]))
                m.shared_experts.up_proj.weight.copy_(torch.from_numpy(w["shared"]["up"]))
                m.shared_experts.down_proj.weight.copy_(torch.from_numpy(w["shared"]["down"]))
            h = hidden_rows(B, D, seed)
            out = m(torch.from_numpy(h)[None]).numpy()[0]
            logits = torch.from_numpy(h) @ m.gate.weight.T
            idx, _ = m.route_tokens_to_experts(logits[None])
        arrays[f"{name}/out"] = out.astype(np.float32)
        arrays[f"{name}/idx"] = np.sort(idx.numpy(), axis=1).astype(np.int64)
        if D <= 256:
            arrays[f"{name}/h"] = h
        meta["cases"].append(dict(name=name, D=D, E=E, K=K, F=F, n_shared=ns, B=B, seed=seed,
                                  scale=scale, h_sha=sha(h), w_sha=weights_sha(w)))
        print(name, "max|out|", float(np.abs(out).max()))
    np.savez_compressed(HERE / "moe_golden.npz", **arrays)
    (HERE / "moe_golden.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
