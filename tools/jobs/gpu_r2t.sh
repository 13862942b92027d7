#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for v in default half g2 g8 l2 na6 na10; do
  for cfg in 1 2 3; do
    if [ $v = default ]; then
      r=$(timeout 300 python tools/time_sweep.py $cfg 2>&1 | grep sweep)
    else
      r=$(HS_LIB=$PWD/variants/libhsweep_$v.so timeout 300 python tools/time_sweep.py $cfg 2>&1 | grep sweep)
    fi
    echo "$v cfg=$cfg $r" >> $O/knobs.log
  done
done
echo done >> $O/knobs.log
