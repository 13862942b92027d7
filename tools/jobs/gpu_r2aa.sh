#!/bin/bash
# multi-right-hand-side sweep: new tests, then timings at C2 / C4 / C3
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "many" > $O/many_tests.log 2>&1; echo "many tests rc=$?" >> $O/rc_aa.txt
timeout 600 python tools/time_many.py 1 1 1 2 4 8 > $O/many_c2.log 2>&1; echo "c2 rc=$?" >> $O/rc_aa.txt
timeout 600 python tools/time_many.py 3 1 1 2 4 8 > $O/many_c4.log 2>&1; echo "c4 rc=$?" >> $O/rc_aa.txt
timeout 900 python tools/time_many.py 2 1 1 2 4 > $O/many_c3.log 2>&1; echo "c3 rc=$?" >> $O/rc_aa.txt
timeout 900 python tools/time_sweep.py 2 > $O/sweep_c3_aa.log 2>&1
echo done >> $O/rc_aa.txt
