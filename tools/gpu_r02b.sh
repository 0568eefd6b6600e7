#!/bin/bash
# r02 session B: fused TP (emulated ranks), Table 1 v2, L2-prefetch sweep, ncu of the step kernel.
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_collective_bench.py -q -x > gpurun_out/pytest_b1.log 2>&1; echo "pytest coll rc $?"; tail -3 gpurun_out/pytest_b1.log
timeout 900 python -m pytest tests/test_gpu_tp_fused.py -q -x -rf > gpurun_out/pytest_b2.log 2>&1; echo "pytest tp rc $?"; tail -15 gpurun_out/pytest_b2.log
timeout 300 python tools/table1_b200.py > gpurun_out/table1_b200.json 2> gpurun_out/table1.log; echo "table1 rc $?"; head -c 1500 gpurun_out/table1.log
timeout 600 python tools/prefetch_ab.py > gpurun_out/prefetch_ab.log 2>&1; echo "pf rc $?"; tail -1 gpurun_out/prefetch_ab.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_step_1024.csv python tools/profile_step_kernel.py 1024 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"; tail -3 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:llama_step -s 1 -c 1 \
  -f -o gpurun_out/prof_step_1024 python tools/profile_step_kernel.py 1024 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"; tail -3 gpurun_out/ncu_full.log
