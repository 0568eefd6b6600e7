#!/bin/bash
# r02 session A: new tests, Table 1 on B200, DSMEM ablation, ncu of the step kernel.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_collective_bench.py tests/test_gpu_persistent.py -q -x > gpurun_out/pytest_a.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_a.log
timeout 300 python tools/table1_b200.py > gpurun_out/table1_b200.json 2> gpurun_out/table1.log; echo "table1 rc $?"
timeout 600 python tools/engine_ab.py --ctx 1024,4096,16384 --engines persistent,persistent_nodsmem,persistent_flat --trace > gpurun_out/engine_ab.log 2>&1; echo "ab rc $?"; tail -1 gpurun_out/engine_ab.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_step_1024.csv python tools/profile_step_kernel.py 1024 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:llama_step -s 1 -c 1 \
  -f -o gpurun_out/prof_step_1024 python tools/profile_step_kernel.py 1024 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
