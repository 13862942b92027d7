#!/bin/bash
# single-RHS X sweep: smaller clusters with 8 segments vs the default C=9, G=7
mkdir -p gpurun_out
O=gpurun_out
for cfg in 2 1 3; do
  echo -n "default C9 G7: " >> $O/layouts_g8.log; python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/layouts_g8.log
  for cg in "8 8" "7 8" "6 8"; do set -- $cg
    echo -n "C$1 G$2: " >> $O/layouts_g8.log; HS_SWEEP_CPC=$1 HS_SWEEP_SEGMENTS=$2 python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/layouts_g8.log
  done
done
echo done >> $O/layouts_g8.log
