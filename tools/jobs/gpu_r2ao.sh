#!/bin/bash
# HS_SWEEP_NA (back-substitution warps; group B = 15 - NA runs the interface GEMV) under the 9-CTA layout
mkdir -p gpurun_out
O=gpurun_out
for cfg in 2 1 3; do
  for v in "" variants/libna7.so variants/libna6.so; do
    echo -n "${v:-default(8)}: " >> $O/na_ab.log
    if [ -z "$v" ]; then python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/na_ab.log; else HS_LIB=$v python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/na_ab.log; fi
  done
done
for v in "" variants/libna7.so; do
  echo "${v:-default(8)}:" >> $O/na_ab.log
  if [ -z "$v" ]; then python tools/time_many.py 3 1 4 2>&1 | grep "x:" >> $O/na_ab.log; else HS_LIB=$v python tools/time_many.py 3 1 4 2>&1 | grep "x:" >> $O/na_ab.log; fi
done
echo done > $O/rc_ao.txt
