#!/bin/bash
# r02 session K: paged KV on the B=1 persistent engine - parity, same-box A/B of the step kernel, paged TPOT.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paged_b1.py tests/test_gpu_persistent.py tests/test_gpu_tp_fused.py -q -x > gpurun_out/pytest_paged_k.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_paged_k.log
timeout 900 bash tools/ab_so.sh tools/scratch/ab/libcfb_A.so tools/scratch/ab/libcfb_B.so \
  "python tools/engine_ab.py --ctx 1024,16384 --engines persistent --steps 50 2>&1 | grep -v "^{"" 1 > gpurun_out/ab_paged_k.log 2>&1; echo "ab rc $?"; cat gpurun_out/ab_paged_k.log
timeout 600 python tools/engine_ab.py --ctx 1024,4096,16384 --engines persistent,persistent_paged,persistent_pagedpm --steps 50 > gpurun_out/paged_tpot_k.log 2>&1; echo "paged rc $?"; cat gpurun_out/paged_tpot_k.log
