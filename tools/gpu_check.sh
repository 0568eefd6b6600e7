#!/bin/bash
# One gpurun session: GPU parity tests, kernel timings, short bench, ncu launch
# list and full captures of the two fused kernels.  Outputs under gpurun_out/.
#   tools/gpu_check.sh [tests|kbench|bench|ncu|full ...]   (default: all)
set -u
mkdir -p gpurun_out
what="${*:-tests kbench bench ncu full}"
for w in $what; do
  case $w in
    tests)  timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
            echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log ;;
    kbench) for c in 1024 16384; do timeout 300 python tools/kbench.py --ctx $c > gpurun_out/kbench_$c.log 2>&1; echo "kbench $c rc $?"; head -c 1500 gpurun_out/kbench_$c.log; echo; done ;;
    bench)  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc $?"; tail -c 2500 gpurun_out/bench.log ;;
    ncu)    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
              --log-file gpurun_out/launches.csv python tools/profile_step.py --ctx 1024 --steps 2 \
              > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?" ;;
    full)   for k in ffn_swiglu mha_split_token lm_head; do
              timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
                -f -o gpurun_out/prof_$k python tools/profile_step.py --ctx 1024 --steps 1 --layers 4 \
                > gpurun_out/ncu_$k.log 2>&1; echo "ncu full $k rc $?"; done ;;
  esac
done
