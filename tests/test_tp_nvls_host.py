"""Host side of the opt-in NVLS sums (tp_fused.NvlsSums) on two gloo ranks
without a GPU: every setup step is agreed over the process group, so a step
that fails on one rank (here cuMulticastCreate on rank 0: no driver on a
CPU host) raises on EVERY rank instead of leaving the others in a barrier."""

from __future__ import annotations

import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_18850_b200.tp_fused import NvlsSums
    try:
        NvlsSums(4096, 0, world=world, rank=rank, group=dist.group.WORLD)
        q.put((rank, "no error"))
    except RuntimeError as exc:
        q.put((rank, str(exc)))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nvls_setup_failure_raises_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert "create/export failed on ranks [0]" in res[r], res
