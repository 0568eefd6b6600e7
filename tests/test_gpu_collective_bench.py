"""The Table-1 latency harness (csrc/collective_bench.cu) computes the right
collective on both channels: ClusterReduce = fp16 sum over ranks (fp32
accumulation in rank order), ClusterGather = rank-ordered concatenation,
every rank holding the result (reference collectives.py:110-203 semantics,
fixtures/table1.csv:4-19 sizes)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("channel", [0, 1])
@pytest.mark.parametrize("op", [0, 3])
@pytest.mark.parametrize("N,kb", [(2, 32), (4, 32), (4, 256), (8, 64), (16, 64)])
def test_collective_bench_results(op, channel, N, kb):
    import torch
    from paper_2508_18850_b200.collective_bench import run_collective
    nbytes = kb * 1024
    rng = np.random.default_rng(N * 1000 + kb + op)
    x = rng.standard_normal((N, nbytes // 2)).astype(np.float16)
    out, ns = run_collective(op, channel, N, x, reps=3)
    if op == 0:
        ref = x.astype(np.float32).sum(0).astype(np.float16)
        for r in range(N):
            np.testing.assert_allclose(out[r].astype(np.float32), ref.astype(np.float32), atol=2e-3, rtol=2e-3)
    else:
        ref = x.reshape(N, N, -1)[np.arange(N), np.arange(N)].reshape(-1)  # rank q's slice q
        for r in range(N):
            assert np.array_equal(out[r], ref)
    assert ns > 0
