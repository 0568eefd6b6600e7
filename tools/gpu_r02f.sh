#!/bin/bash
# r02 session E, call 2: TP shard traces (cluster vs flat), MoE trace, DeepSeek breakdown.
set -u
mkdir -p gpurun_out
timeout 900 python tools/tp_shard_trace.py > gpurun_out/tp_shard_trace.log 2>&1; echo "tp trace rc $?"; grep -v '^\[' gpurun_out/tp_shard_trace.log | cut -c1-400
timeout 300 python tools/moebench.py --pdl > gpurun_out/moebench.log 2>&1; echo "moe rc $?"; tail -3 gpurun_out/moebench.log
timeout 300 python tools/dsbench.py > gpurun_out/dsbench.log 2>&1; echo "ds rc $?"; tail -4 gpurun_out/dsbench.log
