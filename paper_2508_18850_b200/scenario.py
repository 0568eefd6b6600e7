"""Decode-step input contract of the drop-in API.

Field names, shapes, validation errors and the seeded generators follow the
reference's ``scenarios.py`` (``ModelDims`` :30-50, ``DecodeScenario`` :53-98,
``random_mha_scenario`` :112-137, ``random_mla_scenario`` :140-165,
``with_preappended_cache`` :184-207) so that a scenario built here, or one
built by the reference package itself, can be handed to
``run_fused_mha_decode`` unchanged.  The generators reproduce the reference's
draws bit for bit (pinned by ``tests/test_api_host.py`` against the golden
sha256 digests), which is what makes GPU-vs-reference parity runs possible
without shipping the inputs.

Arrays are float32 numpy values; with ``dtype_bytes == 2`` they hold
binary16-representable values (the GPU stores them as fp16).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

from .exceptions import DimensionError, InvalidClusterSize, ShapeMismatch

MHA = "mha"
MLA = "mla"


def _tag(nbytes: int) -> str:
    if nbytes not in (2, 4):
        raise ValueError(f"dtype_bytes must be 2 or 4, got {nbytes}")
    return "f16-emulated" if nbytes == 2 else "f32"


def store_round(a, dtype_bytes: int) -> np.ndarray:
    """Value after a store at ``dtype_bytes`` precision (fp32 compute kept)."""
    a = np.asarray(a, dtype=np.float32)
    if dtype_bytes == 2:
        return a.astype(np.float16).astype(np.float32)
    return a


@dataclass(frozen=True)
class ModelDims:
    batch_size: int
    hidden_dim: int
    n_heads: int
    head_dim: int
    seq_len: int
    kv_lora_rank: int | None = None
    dtype_bytes: int = 4

    def __post_init__(self):
        for name in ("batch_size", "hidden_dim", "n_heads", "head_dim"):
            if getattr(self, name) < 1:
                raise DimensionError(f"{name} must be >= 1")
        if self.seq_len < 0:
            raise DimensionError("seq_len must be >= 0")
        _tag(self.dtype_bytes)

    @property
    def dtype_tag(self) -> str:
        return _tag(self.dtype_bytes)


@dataclass(frozen=True)
class ClusterConfig:
    """Cluster size N (CTAs per head) plus the storage width."""

    n_blocks: int
    smem_capacity_bytes: int | None = None
    dtype_bytes: int = 4

    def __post_init__(self):
        n = self.n_blocks
        if not (1 <= n <= 16) or n & (n - 1):
            raise InvalidClusterSize(
                f"cluster size must be a power of two in [1, 16], got {n}")
        _tag(self.dtype_bytes)
        if self.smem_capacity_bytes is not None and self.smem_capacity_bytes <= 0:
            raise ValueError("smem_capacity_bytes must be positive or None")

    @property
    def dtype_tag(self) -> str:
        return _tag(self.dtype_bytes)


_MHA_SHAPES = {
    "w_qkv": lambda d: (d.n_heads, d.hidden_dim, 3 * d.head_dim),
    "k_cache": lambda d: (d.n_heads, d.seq_len, d.head_dim),
    "v_cache": lambda d: (d.n_heads, d.seq_len, d.head_dim),
}
_MLA_SHAPES = {
    "w_q": lambda d: (d.n_heads, d.hidden_dim, d.head_dim),
    "w_up": lambda d: (d.n_heads, d.head_dim, d.kv_lora_rank),
    "w_kv": lambda d: (d.hidden_dim, d.kv_lora_rank),
    "w_down": lambda d: (d.n_heads, d.kv_lora_rank, d.head_dim),
    "kv_cache": lambda d: (d.seq_len, d.kv_lora_rank),
}


@dataclass
class DecodeScenario:
    """One decode step: B new hidden rows, attention weights, cached K/V."""

    kind: str
    dims: ModelDims
    cluster: ClusterConfig
    hidden: np.ndarray
    seed: int = 0
    w_qkv: np.ndarray | None = None
    k_cache: np.ndarray | None = None
    v_cache: np.ndarray | None = None
    w_q: np.ndarray | None = None
    w_up: np.ndarray | None = None
    w_kv: np.ndarray | None = None
    w_down: np.ndarray | None = None
    kv_cache: np.ndarray | None = None
    w_out: np.ndarray | None = None

    def validate(self) -> None:
        validate_scenario(self)


def _check(arr, shape, name):
    if arr is None:
        raise ShapeMismatch(f"scenario field {name} is missing")
    if tuple(arr.shape) != tuple(shape):
        raise ShapeMismatch(f"scenario field {name} has shape {arr.shape}, expected {shape}")


def validate_scenario(sc) -> None:
    """Shape validation with the reference's error types (works on reference
    scenario objects too: only attributes are used)."""
    d = sc.dims
    if sc.cluster.dtype_bytes != d.dtype_bytes:
        raise ShapeMismatch("cluster dtype_bytes must match dims.dtype_bytes")
    _check(sc.hidden, (d.batch_size, d.hidden_dim), "hidden")
    _check(sc.w_out, (d.n_heads, d.head_dim, d.hidden_dim), "w_out")
    if sc.kind == MHA:
        table = _MHA_SHAPES
    elif sc.kind == MLA:
        if d.kv_lora_rank is None:
            raise DimensionError("mla scenarios require dims.kv_lora_rank")
        table = _MLA_SHAPES
    else:
        raise DimensionError(f"unknown scenario kind {sc.kind!r}")
    for name, shape in table.items():
        _check(getattr(sc, name), shape(d), name)


class _Draws:
    """Seeded N(0,1)*scale draws, float64 -> float32 -> storage rounding."""

    def __init__(self, seed: int, dtype_bytes: int):
        self.rng = np.random.default_rng(seed)
        self.nb = dtype_bytes

    def __call__(self, shape, scale: float) -> np.ndarray:
        return store_round((self.rng.standard_normal(shape) * scale).astype(np.float32), self.nb)


def random_mha_scenario(dims: ModelDims, n_blocks: int = 1, seed: int = 0,
                        smem_capacity_bytes: int | None = None) -> DecodeScenario:
    """Seeded MHA scenario; weights scaled by fan_in^-1/2 (reference draw order)."""
    d = dims
    draw = _Draws(seed, d.dtype_bytes)
    hidden = draw((d.batch_size, d.hidden_dim), 1.0)
    w_qkv = draw((d.n_heads, d.hidden_dim, 3 * d.head_dim), d.hidden_dim ** -0.5)
    w_out = draw((d.n_heads, d.head_dim, d.hidden_dim), d.head_dim ** -0.5)
    k_cache = draw((d.n_heads, d.seq_len, d.head_dim), 1.0)
    v_cache = draw((d.n_heads, d.seq_len, d.head_dim), 1.0)
    sc = DecodeScenario(MHA, d, ClusterConfig(n_blocks, smem_capacity_bytes, d.dtype_bytes),
                        hidden, seed, w_qkv=w_qkv, k_cache=k_cache, v_cache=v_cache,
                        w_out=w_out)
    sc.validate()
    return sc


def random_mla_scenario(dims: ModelDims, n_blocks: int = 1, seed: int = 0,
                        smem_capacity_bytes: int | None = None) -> DecodeScenario:
    """Seeded MLA scenario (needs dims.kv_lora_rank)."""
    d = dims
    if d.kv_lora_rank is None:
        raise DimensionError("random_mla_scenario requires dims.kv_lora_rank")
    r = d.kv_lora_rank
    draw = _Draws(seed, d.dtype_bytes)
    hidden = draw((d.batch_size, d.hidden_dim), 1.0)
    w_q = draw((d.n_heads, d.hidden_dim, d.head_dim), d.hidden_dim ** -0.5)
    w_up = draw((d.n_heads, d.head_dim, r), d.head_dim ** -0.5)
    w_kv = draw((d.hidden_dim, r), d.hidden_dim ** -0.5)
    w_down = draw((d.n_heads, r, d.head_dim), r ** -0.5)
    w_out = draw((d.n_heads, d.head_dim, d.hidden_dim), d.head_dim ** -0.5)
    kv_cache = draw((d.seq_len, r), 1.0)
    sc = DecodeScenario(MLA, d, ClusterConfig(n_blocks, smem_capacity_bytes, d.dtype_bytes),
                        hidden, seed, w_q=w_q, w_up=w_up, w_kv=w_kv, w_down=w_down,
                        kv_cache=kv_cache, w_out=w_out)
    sc.validate()
    return sc


def project_new_kv(sc) -> np.ndarray:
    """New cache rows implied by the hidden states: (n_heads, B, 2H) [K|V] for
    MHA, (B, l) latent rows for MLA; storage-rounded."""
    d = sc.dims
    if sc.kind == MHA:
        rows = [sc.hidden @ sc.w_qkv[i][:, d.head_dim:] for i in range(d.n_heads)]
        return store_round(np.stack(rows), d.dtype_bytes)
    return store_round(sc.hidden @ sc.w_kv, d.dtype_bytes)


def with_preappended_cache(sc):
    """Copy whose cache already holds the new token(s); run it with
    ``append_new_token=False`` to check single counting."""
    d = sc.dims
    dims2 = dataclasses.replace(d, seq_len=d.seq_len + d.batch_size)
    new = project_new_kv(sc)
    if sc.kind == MHA:
        return dataclasses.replace(
            sc, dims=dims2,
            k_cache=np.concatenate([sc.k_cache, new[:, :, :d.head_dim]], axis=1),
            v_cache=np.concatenate([sc.v_cache, new[:, :, d.head_dim:]], axis=1))
    return dataclasses.replace(sc, dims=dims2, kv_cache=np.concatenate([sc.kv_cache, new], 0))
