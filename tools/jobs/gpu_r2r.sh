#!/bin/bash
# level-0 sparse couplings A/B with the 9-CTA layout (bandwidth-bound regime)
mkdir -p gpurun_out
O=gpurun_out
for i in 1 2; do
for cfg in 1 2 3; do
  timeout 300 python tools/time_sweep.py $cfg >> $O/cpl0_ab2.log 2>&1
  HS_SWEEP_CPL0=1 timeout 300 python tools/time_sweep.py $cfg >> $O/cpl0_ab2.log 2>&1
  echo "^ cpl0" >> $O/cpl0_ab2.log
done
done
echo done >> $O/cpl0_ab2.log
