#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for cfg in 2 1; do
  echo "default:" >> $O/fused_tiles.log; python tools/time_fused.py $cfg 2>&1 | grep fused >> $O/fused_tiles.log
  for v in variants/libf_*.so; do
    echo "$v:" >> $O/fused_tiles.log; HS_LIB=$v python tools/time_fused.py $cfg 2>&1 | grep fused >> $O/fused_tiles.log
  done
done
echo done > $O/rc_ah.txt
