#!/bin/bash
# r02 session E: refresh ncu evidence for the current kernels (one GPU, no multi-rank).
set -u
mkdir -p gpurun_out
# step kernel: full set (plain launch) + launch list of 2 eager steps
timeout 600 ncu --set full --clock-control none --import-source on -k regex:llama_step -s 1 -c 1 \
  -o gpurun_out/ncu_step_kernel_e python tools/profile_step_kernel.py 1024 > gpurun_out/ncu_step_e.log 2>&1; echo "ncu step rc $?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_step_e.csv python tools/profile_step_kernel.py 1024 > /dev/null 2>&1; echo "launches rc $?"
# DeepSeek block kernels at 1K: mla_proj / mla_attn / mla_out / moe, one of each (full set)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mla_proj|mla_attn|mla_out|moe_kernel" -s 8 -c 4 \
  -o gpurun_out/ncu_deepseek_e python tools/dsbench.py --contexts 1024 --layers 2 --reps 2 > gpurun_out/ncu_ds_e.log 2>&1; echo "ncu ds rc $?"
ls -la gpurun_out/*.ncu-rep
