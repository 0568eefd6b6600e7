#!/bin/bash
# r02 session O: full GPU suite, smoke, default bench at HEAD (after the B=1 paged KV)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_o.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu_o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_o.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_o.log
timeout 1200 python bench.py > gpurun_out/bench_o.log 2> gpurun_out/bench_o.err; echo "bench rc $?"; tail -c 1500 gpurun_out/bench_o.log
