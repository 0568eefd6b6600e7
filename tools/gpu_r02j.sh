#!/bin/bash
# r02 session J: LM-head evidence (the layered lm_head_kernel: DeepSeek model / layered Llama engine).
set -u
mkdir -p gpurun_out
timeout 300 python tools/profile_lm_head.py > gpurun_out/lm_head_time_j.json 2> gpurun_out/lm_head_time_j.err; echo "lm time rc $?"; cat gpurun_out/lm_head_time_j.json
for m in llama2-7b deepseek-v2-lite; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lm_head -s 1 -c 1 \
    -o gpurun_out/ncu_lm_head_$m python tools/profile_lm_head.py $m > gpurun_out/ncu_lm_head_$m.log 2>&1; echo "ncu $m rc $?"
done
ls -la gpurun_out/*.ncu-rep
