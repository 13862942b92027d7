#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
HS_SWEEP_TRACE=$O/trace_c4_nr1.txt HS_SWEEP_TRACE_NR=1 timeout 600 python tools/time_many.py 3 1 1 > $O/trace_c4_nr1.log 2>&1
HS_SWEEP_TRACE=$O/trace_c4_nr4.txt HS_SWEEP_TRACE_NR=4 timeout 600 python tools/time_many.py 3 1 4 > $O/trace_c4_nr4.log 2>&1
HS_SWEEP_TRACE=$O/trace_c4_nr2.txt HS_SWEEP_TRACE_NR=2 timeout 600 python tools/time_many.py 3 1 2 > $O/trace_c4_nr2.log 2>&1
echo done > $O/rc_ae.txt
