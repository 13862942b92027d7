#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for k in 1 2; do
  for cfg in 2 1; do
    for v in "" variants/libold.so variants/libts.so variants/libts_div.so; do
      echo -n "${v:-default}: " >> $O/ab2.log
      if [ -z "$v" ]; then python tools/time_sweep.py $cfg 2>&1 | tail -1 >> $O/ab2.log; else HS_LIB=$v python tools/time_sweep.py $cfg 2>&1 | tail -1 >> $O/ab2.log; fi
    done
  done
done
echo done > $O/rc_ag.txt
