#!/bin/bash
# C3 sweep layouts with smaller clusters and more segments
mkdir -p gpurun_out
O=gpurun_out
for cg in "16 3" "9 8" "10 7" "8 8" "12 5" "9 7"; do
  set -- $cg
  HS_SWEEP_CPC=$1 HS_SWEEP_SEGMENTS=$2 timeout 300 python tools/time_sweep.py 2 >> $O/sweep_layouts2.log 2>&1
  echo "C=$1 G=$2 rc=$?" >> $O/sweep_layouts2.log
done
for cg in "16 2" "9 4" "8 4" "9 3"; do
  set -- $cg
  HS_SWEEP_CPC=$1 HS_SWEEP_SEGMENTS=$2 timeout 300 python tools/time_sweep.py 1 >> $O/sweep_layouts2.log 2>&1
  echo "C2 C=$1 G=$2 rc=$?" >> $O/sweep_layouts2.log
done
echo done >> $O/sweep_layouts2.log
