#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for v in variants/libg1.so variants/libg2.so variants/libg3.so; do
  echo $v >> $O/sweep3_groups.log
  HS_LIB=$v timeout 900 python tools/time_sweep3.py 2>&1 | tail -n 1 >> $O/sweep3_groups.log
done
echo done > $O/rc_aj.txt
