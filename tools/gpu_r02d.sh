#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python tools/tp_fused_time.py --engine persistent_flat > gpurun_out/tp_fused_time_flat.log 2>&1; echo "tp flat rc $?"; tail -1 gpurun_out/tp_fused_time_flat.log
timeout 300 python tools/skew_probe.py persistent 1024 > gpurun_out/skew.log 2>&1; echo "skew rc $?"; tail -2 gpurun_out/skew.log
