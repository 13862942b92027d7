#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
HS_SWEEP_TRACE=$O/trace_c3.txt timeout 300 python tools/time_sweep.py 2 > $O/trace_c3.log 2>&1
HS_SWEEP_TRACE=$O/trace_c2.txt timeout 300 python tools/time_sweep.py 1 > $O/trace_c2.log 2>&1
for cfg in 1 2 3; do timeout 300 python tools/time_sweep.py $cfg >> $O/sweep_rel.log 2>&1; done
echo done > $O/rc20.txt
