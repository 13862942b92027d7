#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python tools/time_many.py 4 1 1 2 4 > $O/many_c5.log 2>&1; echo "c5 rc=$?" >> $O/rc_am.txt
echo done >> $O/rc_am.txt
