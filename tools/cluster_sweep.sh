#!/bin/bash
# BASELINE.json configs[3]: cluster-size sweep 2/4/8/16 of the split_token
# attention module on the Llama2-7B block at 4K context.  Per N: kernel timing
# (tools/kbench.py, CUDA events) and one ncu pass over the attention launches
# with DRAM bytes, DSMEM bytes (l1tex -> xbar distributed-shared writes) and the
# launch's cluster shape / occupancy.  Outputs under gpurun_out/cluster_sweep/.
set -u
out=gpurun_out/cluster_sweep
mkdir -p $out
avail=$(ncu --query-metrics --chip gb100 2>/dev/null | awk '{print $1}')
want="gpu__time_duration.sum dram__bytes_read.sum dram__bytes_write.sum l1tex__m_l1tex2xbar_write_bytes_mem_dshared.sum l1tex__m_l1tex2xbar_write_bytes_mem_dshared_op_st.sum launch__grid_size launch__cluster_dim_x launch__cluster_max_active launch__occupancy_cluster_pct launch__cluster_scheduling_policy sm__ctas_launched.sum launch__waves_per_multiprocessor"
m=""
for w in $want; do
  base=${w%.sum}
  if echo "$avail" | grep -qx "$base"; then m="$m,$w"; fi
done
m=${m#,}
echo "metrics: $m" > $out/metrics.txt
for n in 2 4 8 16; do
  timeout 200 python tools/kbench.py --ctx 4096 --cluster $n 2>&1 | head -1 > $out/kbench_n$n.json
  timeout 300 ncu --metrics $m --clock-control none -k regex:mha_split_token -s 8 -c 4 --csv \
    --log-file $out/ncu_n$n.csv python tools/kbench.py --ctx 4096 --cluster $n --reps 8 > /dev/null 2>&1
  echo "N=$n $(cat $out/kbench_n$n.json)"
done
