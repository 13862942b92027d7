#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for cfg in 1 3; do
  for g in 2 3 4 5 6 7; do
    HS_SWEEP_CPC=9 HS_SWEEP_SEGMENTS=$g timeout 300 python tools/time_sweep.py $cfg >> $O/sweep_layouts3.log 2>&1
  done
done
for g in 5 6 7; do
  HS_SWEEP_CPC=9 HS_SWEEP_SEGMENTS=$g timeout 300 python tools/time_sweep.py 2 >> $O/sweep_layouts3.log 2>&1
done
for cpc in 4 5 6 7 9; do
  HS_SWEEP_CPC=$cpc timeout 300 python tools/time_sweep.py 0 >> $O/sweep_layouts3.log 2>&1
done
echo done >> $O/sweep_layouts3.log
