#!/bin/bash
# r02 session C: full GPU suite, fused-TP timing on one GPU, DeepSeek breakdown.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python tools/tp_fused_time.py > gpurun_out/tp_fused_time.log 2>&1; echo "tp time rc $?"; tail -1 gpurun_out/tp_fused_time.log
timeout 300 python tools/dsbench.py > gpurun_out/dsbench.log 2>&1; echo "ds rc $?"; tail -3 gpurun_out/dsbench.log
