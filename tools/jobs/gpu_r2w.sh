#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
HS_SWEEP_TRACE=$O/trace_c3.txt timeout 300 python tools/time_sweep.py 2 > $O/trace_c3.log 2>&1
HS_SWEEP_TRACE=$O/trace_c2.txt timeout 300 python tools/time_sweep.py 1 > $O/trace_c2.log 2>&1
echo done > $O/rc19.txt
