"""paper_2508_18850_b200 — B200-native ClusterFusion decode-step hot path.

Drop-in for the reference ``clusterdec`` package's fused-dataflow API
(``/root/reference/pkg/src/clusterdec/__init__.py:11-62``): the same
scenario containers, generators, result type, ledger/traffic model and error
classes, with the dataflows executed by hand-written sm_100a kernels
(``csrc/``, built into ``libcfb.so``, C ABI in ``include/cfb.h``).
There is no CPU fallback.
"""

from .exceptions import (BufferError, DimensionError, FixtureError, InvalidClusterSize,  # noqa: F401
                         OutOfBounds, ShapeMismatch, SimulationError, SmemOverflow)
from .fused import (DATAFLOW_KINDS, FUSED_MLA, MERGED, SPLIT_HEAD, SPLIT_TOKEN,  # noqa: F401
                    TWO_PASS, DecodeResult, cluster_collective, run_dataflow,
                    run_fused_mha_decode, sequence_segments, validate_partitioning)
from .devcache import PreparedScenario, clear_device_cache, prepare  # noqa: F401
from .mla import run_fused_mla_decode, run_splithead_decode  # noqa: F401
from .moe import MoeWeights, pack_moe, run_moe_decode  # noqa: F401
from .ledger import (CollectiveTrace, StageTrace, TrafficBreakdown, TrafficEntry,  # noqa: F401
                     TrafficEvent, TrafficLedger, dataflow_traffic, reconcile_traffic,
                     traffic_gather, traffic_reduce)
from .scenario import (MHA, MLA, ClusterConfig, DecodeScenario, ModelDims,  # noqa: F401
                       project_new_kv, random_mha_scenario, random_mla_scenario,
                       with_preappended_cache)

__version__ = "0.2.0"
