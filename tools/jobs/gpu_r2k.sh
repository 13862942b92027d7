#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "3d or pml3d or C5 or exact or factor or dense" > $O/gputest11.log 2>&1; echo "gputest rc=$?" >> $O/rc11.txt
for i in 1 2; do
HS_LIB=$PWD/variants/libhsweep_bar1.so timeout 600 python tools/time_sweep3.py >> $O/bar_ab.log 2>&1
echo "^ one counter" >> $O/bar_ab.log
timeout 600 python tools/time_sweep3.py >> $O/bar_ab.log 2>&1
echo "^ 8 counters" >> $O/bar_ab.log
done
echo done >> $O/rc11.txt
