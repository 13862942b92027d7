#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
L=$PWD/variants/libhsweep_g16.so
for cg in "9 7" "6 12" "6 10" "7 9" "5 14" "4 16" "8 8"; do
  set -- $cg
  for cfg in 2 1; do
    r=$(HS_LIB=$L HS_SWEEP_CPC=$1 HS_SWEEP_SEGMENTS=$2 timeout 300 python tools/time_sweep.py $cfg 2>&1 | grep sweep)
    echo "C=$1 G=$2 cfg=$cfg $r" >> $O/knobs2.log
  done
done
echo done >> $O/knobs2.log
