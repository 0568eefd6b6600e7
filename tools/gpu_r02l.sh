#!/bin/bash
# r02 session L: paged B=1 TPOT, shuffled vs in-order pages
set -u
mkdir -p gpurun_out
timeout 600 python tools/engine_ab.py --ctx 1024,16384 --engines persistent,persistent_pagedseq,persistent_paged --steps 50 > gpurun_out/paged_tpot_l.log 2>&1; echo "rc $?"; cat gpurun_out/paged_tpot_l.log
