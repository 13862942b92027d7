#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "many" > $O/many3d_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_al.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_al.log 2>&1; echo "gputest rc=$?" >> $O/rc_al.txt
timeout 900 python tools/time_sweep3.py > $O/sweep3_al.log 2>&1
echo done >> $O/rc_al.txt
