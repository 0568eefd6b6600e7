#!/bin/bash
# r02 session N: paged producer loop A/B (B: shuffles every trip, C: only on issuing trips) + paged parity with C
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_paged_b1.py tests/test_gpu_persistent.py tests/test_gpu_tp_fused.py tests/test_gpu_parity_long.py -q -x > gpurun_out/pytest_paged_n.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_paged_n.log
timeout 900 bash tools/ab_so.sh tools/scratch/ab/libcfb_E.so tools/scratch/ab/libcfb_F.so \
  "python tools/engine_ab.py --ctx 1024,16384 --engines persistent,persistent_paged,persistent_pagedseq --steps 50 2>&1 | grep -v '^{'" 2 > gpurun_out/ab_paged_n.log 2>&1; echo "ab rc $?"; cat gpurun_out/ab_paged_n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke_n.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_n.log
