#!/bin/bash
# Cluster occupancy evidence for the split_token attention module (Llama2-7B
# block, 4K context) at cluster sizes 2/4/8/16: one ncu capture per N with the
# LaunchStats + Occupancy sections (cluster shape, max active clusters, cluster
# occupancy) plus DRAM / DSMEM bytes.  Reports under gpurun_out/cluster_occ/.
set -u
out=gpurun_out/cluster_occ
mkdir -p $out
for n in 2 4 8 16; do
  timeout 300 ncu --section LaunchStats --section Occupancy --section SpeedOfLight \
    --metrics dram__bytes_read.sum,l1tex__m_l1tex2xbar_write_bytes_mem_dshared.sum \
    --clock-control none -k regex:mha_split_token -s 8 -c 1 -o $out/occ_n$n -f \
    python tools/kbench.py --ctx 4096 --cluster $n --reps 2 > $out/log_n$n.txt 2>&1
  echo "N=$n rc=$?"
done
