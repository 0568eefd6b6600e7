#!/bin/bash
# A/B two builds of libcfb.so on ONE box, alternating: tools/ab_so.sh A.so B.so "<command>" [rounds]
set -u
A=$1; B=$2; CMD=$3; R=${4:-2}
LIB=paper_2508_18850_b200/libcfb.so
cp $LIB /tmp/libcfb_orig.so
for r in $(seq 1 $R); do
  for v in A B; do
    if [ $v = A ]; then cp $A $LIB; else cp $B $LIB; fi
    echo "== $v round $r"; bash -c "$CMD"
  done
done
cp /tmp/libcfb_orig.so $LIB
