"""Drop-in API device residency (devcache.py): a cached or prepared call
equals an uncached one, repeated calls do not re-upload, and arrays mutated in
place are never served stale."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2508_18850_b200 as cfb
from oracle import clusterdec_port as cp
from paper_2508_18850_b200.devcache import CACHE

pytestmark = pytest.mark.gpu


def test_cached_and_prepared_equal_uncached():
    cfb.clear_device_cache()
    dims = cfb.ModelDims(1, 1024, 8, 128, 300, dtype_bytes=2)
    sc = cfb.random_mha_scenario(dims, n_blocks=4, seed=5)
    first = cfb.run_fused_mha_decode(sc)          # miss: uploads
    m0 = CACHE.misses
    again = cfb.run_fused_mha_decode(sc)          # hit: nothing re-uploaded
    assert CACHE.misses == m0 and CACHE.hits >= 4
    prep = cfb.prepare(sc)
    viaprep = cfb.run_fused_mha_decode(prep)
    assert np.array_equal(first.output, again.output)
    assert np.array_equal(first.output, viaprep.output)
    assert first.stage_traffic == viaprep.stage_traffic
    # a new hidden block through the prepared handle: only the activation changes
    h2 = np.ascontiguousarray(sc.hidden[:, ::-1])
    r2 = cfb.run_fused_mha_decode(prep.with_hidden(h2))
    ref = cp.dense_mha(h2, sc.w_qkv, sc.w_out, sc.k_cache, sc.v_cache)
    assert float(np.max(np.abs(r2.output - ref))) <= 2e-2


def test_mutated_arrays_are_not_served_stale():
    cfb.clear_device_cache()
    dims = cfb.ModelDims(1, 512, 4, 64, 100, dtype_bytes=4)
    sc = cfb.random_mha_scenario(dims, n_blocks=2, seed=6)
    a = cfb.run_fused_mha_decode(sc).output
    sc.w_out[1, 3, 7] += 0.5           # in-place edits of a cached weight
    sc.k_cache[0, 10] *= -1.0          # ... and of the cache
    b = cfb.run_fused_mha_decode(sc).output
    ref = cp.dense_mha(sc.hidden, sc.w_qkv, sc.w_out, sc.k_cache, sc.v_cache)
    assert not np.array_equal(a, b)
    np.testing.assert_allclose(b, ref, atol=1e-4)


def test_mla_prepared_equals_scenario():
    cfb.clear_device_cache()
    dims = cfb.ModelDims(1, 256, 2, 32, 40, 64, dtype_bytes=2)
    sc = cfb.random_mla_scenario(dims, n_blocks=2, seed=1)
    a = cfb.run_fused_mla_decode(sc)
    b = cfb.run_fused_mla_decode(cfb.prepare(sc))
    assert np.array_equal(a.output, b.output)
