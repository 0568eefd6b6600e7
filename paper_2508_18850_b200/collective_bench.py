"""Host side of the Table-1 harness (csrc/collective_bench.cu): on-chip
(DSMEM bulk copies) vs off-chip (global memory) ClusterReduce /
ClusterGather latency on one cluster, operands and results in shared memory.
Reference: fixtures/table1.csv:4-19."""

from __future__ import annotations

import numpy as np

from . import _native

OPS = {"reduce": 0, "gather": 3}
CHANNELS = {"on_chip": 0, "off_chip": 1}
SCRATCH_BYTES = 1 << 20


def _bufs(torch, n_out_halves):
    out = torch.zeros(n_out_halves, dtype=torch.float16, device="cuda")
    scratch = torch.zeros(SCRATCH_BYTES // 2, dtype=torch.float16, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    ns = torch.zeros(1, dtype=torch.int64, device="cuda")
    return out, scratch, ctr, ns


def run_collective(op: int, channel: int, N: int, x: np.ndarray, reps: int = 3):
    """Validation run.  x [N][n] fp16 (reduce: every rank's full vector;
    gather: rank q contributes slice q of x[q] reshaped [N][n/N]).  Returns
    (out [N][n] fp16, mean ns per collective)."""
    import torch
    _native.require_cuda()
    L = _native.lib()
    N_, n = x.shape
    assert N_ == N
    if op == 3:
        src = np.stack([x[q].reshape(N, -1)[q] for q in range(N)]).reshape(-1)
    else:
        src = x.reshape(-1)
    din = torch.from_numpy(np.ascontiguousarray(src)).cuda()
    out, scratch, ctr, ns = _bufs(torch, N * n)
    _native.check(L.cfb_collective_bench(op, channel, N, n * 2, reps, 1, din.data_ptr(), out.data_ptr(),
                                         scratch.data_ptr(), ctr.data_ptr(), ns.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.view(N, n).cpu().numpy(), int(ns.item())


def time_collective(op: str, channel: str, N: int, kb: int, reps: int = 200, launches: int = 20):
    """(in-kernel ns per collective, event-timed us per one-collective launch)
    for one Table-1 cell; timing mode (no HBM traffic)."""
    import torch
    L = _native.lib()
    out, scratch, ctr, ns = _bufs(torch, 8)
    st = torch.cuda.current_stream().cuda_stream

    def launch(r):
        _native.check(L.cfb_collective_bench(OPS[op], CHANNELS[channel], N, kb * 1024, r, 0, None,
                                             out.data_ptr(), scratch.data_ptr(), ctr.data_ptr(),
                                             ns.data_ptr(), st))
    for _ in range(3):
        launch(reps)
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        launch(reps)
        torch.cuda.synchronize()
        v = int(ns.item())
        best = v if best is None else min(best, v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(launches):
        launch(1)
    e1.record()
    torch.cuda.synchronize()
    return best, e0.elapsed_time(e1) * 1e3 / launches
