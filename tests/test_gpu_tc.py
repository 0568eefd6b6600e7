"""Batch-16 projections on tcgen05 (csrc/tc_gemm.cu) against an fp32 numpy
reference of the same contraction on identical fp16-valued inputs
(tolerance: max-abs 2e-2 and max-rel 1e-3 of max|y| - fp32 TMEM accumulation,
fixed-point split-K sums)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle.llama_port import f16
from paper_2508_18850_b200.tc import TcProjection, pack_umma, run_projection_b16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,K", [(128, 64), (256, 128), (384, 1024), (4096, 4096), (4096, 11008)])
def test_tc_projection_matches_fp32(M, K):
    rng = np.random.default_rng(M + K)
    w = f16(rng.standard_normal((M, K)) * K ** -0.5)
    x = f16(rng.standard_normal((16, K)))
    y = run_projection_b16(w, x)
    ref = x @ w.T
    err = float(np.max(np.abs(y - ref)))
    assert err <= 2e-2 and err <= 1e-3 * max(1.0, float(np.max(np.abs(ref)))), (M, K, err)


def test_tc_projection_repeat_and_layout():
    """Repeated launches re-zero the accumulator; the packing is a pure permutation."""
    import torch
    rng = np.random.default_rng(0)
    w = f16(rng.standard_normal((256, 128)))
    x = f16(rng.standard_normal((16, 128)))
    proj = TcProjection(w)
    xt = torch.from_numpy(x).cuda().half()
    y = torch.empty(16, 256, device="cuda")
    outs = []
    for _ in range(3):
        proj.launch(xt, y)
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy().copy())
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()
    wp = pack_umma(torch.from_numpy(w).half())
    assert sorted(wp.flatten().float().tolist()) == sorted(torch.from_numpy(w).half().flatten().float().tolist())


@pytest.mark.parametrize("D,F", [(512, 1408), (4096, 11008)])
def test_tc_ffn_b16_matches_oracle(D, F):
    """Batch-16 FFN block (RMSNorm -> SwiGLU -> residual) vs oracle/llama_port.ffn_block."""
    import torch
    from oracle import llama_port as lp
    from paper_2508_18850_b200.tc import TcFfnB16
    rng = np.random.default_rng(D)
    x = rng.standard_normal((16, D)).astype(np.float32)
    g = f16(1 + 0.1 * rng.standard_normal(D))
    w1 = f16(rng.standard_normal((F, D)) * D ** -0.5)
    w2 = f16(rng.standard_normal((F, D)) * D ** -0.5)
    w3 = f16(rng.standard_normal((D, F)) * F ** -0.5)
    ffn = TcFfnB16(w1, w2, w3, g, eps=1e-5)
    r = torch.from_numpy(x).cuda()
    ffn.launch(r)
    torch.cuda.synchronize()
    got = r.cpu().numpy()
    ref = x + lp.ffn_block(x, g, w1, w2, w3, 1e-5)
    err = float(np.max(np.abs(got - ref)))
    assert err <= 2e-2 and err / float(np.max(np.abs(ref))) <= 1e-2, err


@pytest.mark.parametrize("M,K", [(256, 128), (384, 1024), (4096, 4096), (4096, 11008), (22016, 4096)])
def test_tc_projection_cta_pairs_match_fp32(M, K):
    """CFB_TC_PAIR: CTA pairs multicast each activation block into both CTAs
    (odd tile counts, e.g. M = 384, fall back to single CTAs)."""
    rng = np.random.default_rng(M * 7 + K)
    w = f16(rng.standard_normal((M, K)) * K ** -0.5)
    x = f16(rng.standard_normal((16, K)))
    y = run_projection_b16(w, x, pair=True)
    ref = x @ w.T
    err = float(np.max(np.abs(y - ref)))
    assert err <= 2e-2 and err <= 1e-3 * max(1.0, float(np.max(np.abs(ref)))), (M, K, err)


@pytest.mark.parametrize("D,F", [(512, 1408), (4096, 11008)])
def test_tc_ffn_b16_cta_pairs_match_oracle(D, F):
    """The batch-16 FFN on CTA pairs (multicast activations) vs the oracle,
    repeated launches on the same residual stream."""
    import torch
    from oracle import llama_port as lp
    from paper_2508_18850_b200.tc import TcFfnB16
    rng = np.random.default_rng(D + 1)
    x = rng.standard_normal((16, D)).astype(np.float32)
    g = f16(1 + 0.1 * rng.standard_normal(D))
    w1 = f16(rng.standard_normal((F, D)) * D ** -0.5)
    w2 = f16(rng.standard_normal((F, D)) * D ** -0.5)
    w3 = f16(rng.standard_normal((D, F)) * F ** -0.5)
    ffn = TcFfnB16(w1, w2, w3, g, eps=1e-5)
    r = torch.from_numpy(x).cuda()
    ref = x
    for _ in range(2):
        ffn.launch(r, pdl=True, pair=True)
        ref = ref + lp.ffn_block(ref, g, w1, w2, w3, 1e-5)
    torch.cuda.synchronize()
    got = r.cpu().numpy()
    err = float(np.max(np.abs(got - ref)))
    assert err <= 2e-2 and err / float(np.max(np.abs(ref))) <= 1e-2, err
