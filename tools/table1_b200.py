"""Re-measure the paper's Table 1 on B200: ClusterReduce / ClusterGather,
on-chip (DSMEM) vs off-chip (global memory), cluster size 4, 32-256 KB
(fixtures/table1.csv:4-19), plus the cluster sizes 2/8/16.
    python tools/table1_b200.py > gpurun_out/table1_b200.json"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_18850_b200.collective_bench import time_collective  # noqa: E402

H100 = {("reduce", 32): (8.03, 6.77), ("reduce", 64): (9.01, 6.61), ("reduce", 128): (14.95, 7.42),
        ("reduce", 256): (22.44, 9.17), ("gather", 32): (6.26, 3.90), ("gather", 64): (6.27, 4.12),
        ("gather", 128): (6.31, 4.39), ("gather", 256): (6.61, 4.15)}
rows = []
for N in (4, 2, 8, 16):
    for op in ("reduce", "gather"):
        for kb in (32, 64, 128, 256):
            r = {"operation": op, "size_kb": kb, "cluster": N}
            for ch in ("off_chip", "on_chip"):
                ns, us_launch = time_collective(op, ch, N, kb)
                r[f"{ch}_us"] = round(ns / 1e3, 3)
                r[f"{ch}_launch_us"] = round(us_launch, 3)
            r["speedup"] = round(r["off_chip_us"] / r["on_chip_us"], 2)
            if N == 4:
                r["h100_off_chip_us"], r["h100_on_chip_us"] = H100[(op, kb)]
                r["h100_speedup"] = round(H100[(op, kb)][0] / H100[(op, kb)][1], 2)
            rows.append(r)
            print(json.dumps(r), file=sys.stderr, flush=True)
print(json.dumps({"what": "B200 Table 1: in-kernel mean time per collective (200 back-to-back reps, "
                          "globaltimer on rank 0) and event-timed single-collective launch",
                  "rows": rows}, indent=1))
