#!/bin/bash
# r02 session I: full GPU suite, smoke, default bench (after the MLA grid / CTA-pair changes).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_i.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu_i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_i.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_i.log
timeout 1200 python bench.py > gpurun_out/bench_i.log 2> gpurun_out/bench_i.err; echo "bench rc $?"; tail -c 3000 gpurun_out/bench_i.log
