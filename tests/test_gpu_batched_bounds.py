"""Batch-16 position bounds (advisor finding): a step that would append past a
sequence's contiguous cache or its reserved pages is refused on the host;
unassigned block-table entries are -1, never page 0."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2508_18850_b200.batched import BatchedLlama
from paper_2508_18850_b200.exceptions import DimensionError
from paper_2508_18850_b200.llama import LlamaConfig

pytestmark = pytest.mark.gpu

CFG = LlamaConfig(n_layers=1, hidden=256, n_heads=2, head_dim=128, inter=384, vocab=256)


def test_contiguous_cache_full_is_refused():
    import torch
    m = BatchedLlama.random(CFG, cache_cap=130, seed=1)
    m.set_positions([127] * 16)
    m.step()
    m.step()  # rows 127, 128 written
    torch.cuda.synchronize()
    m.step()  # row 129 = cap - 1: still fits
    with pytest.raises(DimensionError):
        m.step()  # row 130 would be past the cache
    with pytest.raises(DimensionError):
        m.set_positions([130] * 16)


def test_paged_needs_reserved_pages_and_table_is_minus_one():
    import torch
    m = BatchedLlama.random_paged(CFG, max_len=512, seed=2)
    m.random_head(CFG.vocab)
    pool = m.pool
    pool.release(3)
    assert (pool.table[3].cpu().numpy() == -1).all()
    pos = [126] * 16
    m.set_positions(pos)  # reserves the page of position 126 for seq 3 again
    assert pool.capacity(3) == 128
    m.decode_step()
    m.decode_step()  # 126, 127
    torch.cuda.synchronize()
    with pytest.raises(DimensionError):
        m.decode_step()  # 128 needs page 1 of seq 3: not reserved
    m.reserve(4)
    m.decode_step()
    torch.cuda.synchronize()
    assert m.pos.cpu().tolist() == [129] * 16
    assert bool(((m.tokens >= 0) & (m.tokens < CFG.vocab)).all())


def test_captured_replay_stops_at_max_len():
    import torch
    m = BatchedLlama.random_paged(CFG, max_len=256, seed=3)
    m.random_head(CFG.vocab)
    m.set_positions([253] * 16)
    m.decode_step()
    torch.cuda.synchronize()
    m.set_positions([253] * 16)
    m.capture_decode()
    m.replay()
    m.replay()  # 253, 254 -> next is 255 (last of max_len 256)
    m.replay()
    with pytest.raises(DimensionError):
        m.replay()
    torch.cuda.synchronize()
    assert np.asarray(m.pos.cpu()).tolist() == [256] * 16
