#!/bin/bash
# r02 session Q: DRAM bytes + duration of the step kernel, contiguous vs paged KV, at 16K (one launch each)
set -u
mkdir -p gpurun_out
for v in contig paged; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:llama_step --launch-skip 1 -c 1 --csv --log-file gpurun_out/ncu_step16k_$v.csv \
    python tools/profile_step_kernel.py 16384 persistent $v > gpurun_out/ncu_step16k_$v.log 2>&1; echo "$v rc $?"
  grep -E "dram__bytes|gpu__time" gpurun_out/ncu_step16k_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
