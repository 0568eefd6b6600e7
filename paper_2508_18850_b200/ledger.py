"""DSMEM traffic ledger and its closed-form model (host logic of the drop-in API).

The GPU kernels execute a *static* collective schedule, so the ledger a
``DecodeResult`` carries is emitted from that schedule event by event in the
order the reference simulator records them (``simcore.py:144-184``,
``collectives.py:110-203``); the kernels additionally count the bytes they
actually pushed through DSMEM (``cfb_mha_args.traffic``) and the API checks
the two agree.  Closed forms follow ``analysis.py:64-263``.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

from .exceptions import DimensionError

DSMEM, GLOBAL = "dsmem", "global"
REDUCE, GATHER = "reduce", "gather"


@dataclass(frozen=True)
class TrafficEvent:
    round: int
    src_rank: int
    dst_rank: int
    nbytes: int
    channel: str


class TrafficLedger:
    """Ordered list of data movements (one event per message)."""

    def __init__(self):
        self.events: list[TrafficEvent] = []

    def record(self, round: int, src_rank: int, dst_rank: int, nbytes: int, channel: str) -> None:  # noqa: A002
        if nbytes <= 0:
            raise ValueError("ledger events must move a positive number of bytes")
        if channel not in (DSMEM, GLOBAL):
            raise ValueError(f"unknown channel {channel!r}")
        self.events.append(TrafficEvent(round, src_rank, dst_rank, nbytes, channel))

    def mark(self) -> int:
        return len(self.events)

    def bytes_since(self, mark: int, channel: str = DSMEM) -> int:
        return sum(e.nbytes for e in self.events[mark:] if e.channel == channel)

    def channel_bytes(self, channel: str = DSMEM) -> int:
        return sum(e.nbytes for e in self.events if e.channel == channel)

    def __len__(self) -> int:
        return len(self.events)


@dataclass(frozen=True)
class CollectiveTrace:
    primitive: str
    payload_bytes: int
    rounds: int
    dsmem_bytes: int


@dataclass(frozen=True)
class StageTrace:
    stage: str
    head: int
    trace: CollectiveTrace


def log2_exact(n: int) -> int:
    if n < 1 or n & (n - 1):
        raise DimensionError(f"cluster size must be a power of two, got {n}")
    return n.bit_length() - 1


def traffic_reduce(size_bytes: int, n_blocks: int) -> int:
    """Channel bytes of one ClusterReduce: size * log2(N) * N."""
    if size_bytes < 0:
        raise ValueError("size_bytes must be >= 0")
    return size_bytes * log2_exact(n_blocks) * n_blocks


def traffic_gather(size_bytes: int, n_blocks: int) -> int:
    """Channel bytes of one ClusterGather: size * (N - 1) * N."""
    if size_bytes < 0:
        raise ValueError("size_bytes must be >= 0")
    log2_exact(n_blocks)
    return size_bytes * (n_blocks - 1) * n_blocks


def emit_reduce(ledger: TrafficLedger, n: int, payload: int) -> CollectiveTrace:
    """Events of one exponential-stride reduce (collectives.py:110-157)."""
    rounds = log2_exact(n)
    for r in range(rounds):
        s = 1 << r
        for b in range(n):
            ledger.record(r, b, (b + s) % n, payload, DSMEM)
    return CollectiveTrace(REDUCE, payload, rounds, payload * rounds * n)


def emit_gather(ledger: TrafficLedger, n: int, seg: int) -> CollectiveTrace:
    """Events of one doubling-prefix gather (collectives.py:160-203)."""
    rounds = log2_exact(n)
    total = 0
    for r in range(rounds):
        s = 1 << r
        for b in range(n):
            ledger.record(r, b, (b + s) % n, seg * s, DSMEM)
            total += seg * s
    return CollectiveTrace(GATHER, seg, rounds, total)


def emit_oneshot(ledger: TrafficLedger, n: int, payload: int, primitive: str) -> CollectiveTrace:
    """Events of one single-round all-to-all push (the decode engine's
    latency-optimal ClusterGather / fused softmax-merge, CFB_ONESHOT): every
    block sends its payload to each of the N-1 peers in round 0.  A gather
    moves the same total bytes as the doubling schedule, N(N-1)*payload."""
    log2_exact(n)
    for b in range(n):
        for d in range(1, n):
            ledger.record(0, b, (b + d) % n, payload, DSMEM)
    return CollectiveTrace(primitive, payload, 1 if n > 1 else 0, payload * (n - 1) * n)


ONESHOT_MERGE = "oneshot_merge"


@dataclass(frozen=True)
class TrafficEntry:
    stage: str
    primitive: str
    payload_bytes: int
    analytical_bytes: int
    is_stats: bool = False
    measured_bytes: int | None = None

    @property
    def reconciled(self) -> bool:
        return self.measured_bytes == self.analytical_bytes


@dataclass
class TrafficBreakdown:
    kind: str
    n_blocks: int
    n_clusters: int
    entries: list = field(default_factory=list)
    swapped_form_bytes: int | None = None

    @property
    def headline_bytes(self) -> int:
        return sum(e.analytical_bytes for e in self.entries if not e.is_stats)

    @property
    def stats_bytes(self) -> int:
        return sum(e.analytical_bytes for e in self.entries if e.is_stats)

    @property
    def total_bytes(self) -> int:
        return self.headline_bytes + self.stats_bytes

    @property
    def model_total_bytes(self) -> int:
        return self.total_bytes * self.n_clusters

    @property
    def reconciled(self) -> bool:
        return all(e.reconciled for e in self.entries)


def _entry(stage, prim, payload, n, is_stats=False) -> TrafficEntry:
    f = traffic_reduce if prim == REDUCE else traffic_gather  # one-shot merge: N(N-1)*payload
    return TrafficEntry(stage, prim, payload, f(payload, n), is_stats)


def dataflow_traffic(kind: str, dims, n_blocks: int, stats_mode: str = "two_pass") -> TrafficBreakdown:
    """Per-cluster analytical DSMEM budget (analysis.py:178-238)."""
    if kind == "split_token_mha":
        kind = "split_token"
    if kind not in ("split_token", "fused_mla", "split_head"):
        raise DimensionError(f"unknown dataflow kind {kind!r}")
    log2_exact(n_blocks)
    nb, B = dims.dtype_bytes, dims.batch_size
    if dims.head_dim % n_blocks:
        raise DimensionError(f"head_dim {dims.head_dim} not divisible by {n_blocks}")
    h = dims.head_dim // n_blocks
    if stats_mode == "oneshot":
        if kind != "split_token":
            raise DimensionError("stats_mode='oneshot' is implemented for split_token")
        h = dims.head_dim // n_blocks
        return TrafficBreakdown(kind, n_blocks, dims.n_heads, [
            _entry("qkv_gather", GATHER, B * 3 * h * nb, n_blocks),
            _entry("attn_state_merge", ONESHOT_MERGE, (2 * B + B * dims.head_dim) * 4, n_blocks)])
    if stats_mode == "merged":
        stats = [_entry("stats_merge_reduce", REDUCE, 2 * B * nb, n_blocks, True)]
    else:
        stats = [_entry("stats_max_reduce", REDUCE, B * nb, n_blocks, True),
                 _entry("stats_sum_reduce", REDUCE, B * nb, n_blocks, True)]
    swapped = None
    if kind == "split_token":
        entries = [_entry("qkv_gather", GATHER, B * 3 * h * nb, n_blocks), *stats,
                   _entry("attn_out_reduce", REDUCE, B * dims.head_dim * nb, n_blocks)]
        swapped = (traffic_reduce(B * 3 * h * nb, n_blocks)
                   + traffic_gather(B * dims.head_dim * nb, n_blocks))
    elif kind == "fused_mla":
        if dims.kv_lora_rank is None or dims.kv_lora_rank % n_blocks:
            raise DimensionError("fused_mla needs kv_lora_rank divisible by cluster size")
        rs = dims.kv_lora_rank // n_blocks
        entries = [_entry("q_proj_gather", GATHER, B * h * nb, n_blocks),
                   _entry("latent_kv_gather", GATHER, B * rs * nb, n_blocks),
                   _entry("absorbed_q_gather", GATHER, B * rs * nb, n_blocks), *stats,
                   _entry("attn_out_reduce", REDUCE, B * dims.kv_lora_rank * nb, n_blocks),
                   _entry("down_proj_reduce", REDUCE, B * dims.head_dim * nb, n_blocks)]
    else:
        att = dims.seq_len + B
        entries = [_entry("score_reduce", REDUCE, B * att * nb, n_blocks),
                   _entry("out_proj_reduce", REDUCE, B * dims.hidden_dim * nb, n_blocks)]
    return TrafficBreakdown(kind, n_blocks, dims.n_heads, entries, swapped)


def reconcile_traffic(kind: str, result, dims, stats_mode: str = "two_pass") -> TrafficBreakdown:
    """Fill measured per-cluster bytes from a result's stage tallies
    (analysis.py:241-263); unmodelled stages raise DimensionError."""
    bd = dataflow_traffic(kind, dims, result.n_blocks, stats_mode)
    heads = result.n_clusters
    measured = dict(result.stage_traffic)
    out = []
    for e in bd.entries:
        tot = measured.pop(e.stage, 0)
        per = tot // heads if heads > 0 and tot % heads == 0 else tot
        out.append(replace(e, measured_bytes=per))
    if measured:
        raise DimensionError("run recorded unmodeled stages: " + ", ".join(sorted(measured)))
    bd.entries = out
    return bd
