#!/bin/bash
# r02 session E: checkpoint re-validation (full GPU suite + smoke + default bench line).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?"; tail -c 3000 gpurun_out/bench.log
