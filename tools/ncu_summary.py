"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py rep  <file.ncu-rep> [--bytes ALGO_BYTES]   -> JSON of key metrics
    python tools/ncu_summary.py launches <launches.csv>                    -> per-kernel time share
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "launch__grid_size", "launch__cluster_size", "launch__cluster_max_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_dshared.sum",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
         "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6}


def rep(path, algo_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    d[k + " [SI]"] = v * SCALE[u]
                else:
                    d[k] = v
        t = d.get("gpu__time_duration.sum [SI]")
        traffic = d.get("dram__bytes_read.sum [SI]", 0) + d.get("dram__bytes_write.sum [SI]", 0)
        d["traffic_bytes"] = traffic
        if algo_bytes and t:
            d["algorithmic_bytes"] = algo_bytes
            d["achieved_GBps_algorithmic"] = algo_bytes / t / 1e9
            d["traffic_over_algorithmic"] = traffic / algo_bytes
        res.append(d)
    return res


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"]
        if "at::" in name or "distribution" in name:
            continue  # torch setup kernels (weight init), not part of the step
        short = name.split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", "")) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        agg[short][0] += 1
        agg[short][1] += v
    tot = sum(v[1] for v in agg.values())
    return {"total_us": round(tot, 1),
            "kernels": {k: {"launches": n, "total_us": round(t, 1), "avg_us": round(t / n, 2),
                            "share": round(t / tot, 4)} for k, (n, t) in
                        sorted(agg.items(), key=lambda kv: -kv[1][1])}}


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        ab = float(sys.argv[sys.argv.index("--bytes") + 1]) if "--bytes" in sys.argv else None
        print(json.dumps(rep(sys.argv[2], ab), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2]), indent=1))
