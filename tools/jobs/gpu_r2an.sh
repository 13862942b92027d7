#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python tools/time_many.py 4 1 1 2 4 > $O/many_c5_seg4.log 2>&1; echo "seg4 rc=$?" >> $O/rc_an.txt
HS_LIB=variants/libseg8.so timeout 900 python tools/time_sweep3.py 2>&1 | tail -n 1 > $O/sweep3_seg8.log
HS_LIB=variants/libseg2.so timeout 900 python tools/time_sweep3.py 2>&1 | tail -n 1 > $O/sweep3_seg2.log
timeout 1200 python -m pytest tests -q -x -m gpu -k "3d or exact or factorize or line1d or C5 or deterministic or many" > $O/tests3d_an.log 2>&1; echo "tests3d rc=$?" >> $O/rc_an.txt
echo done >> $O/rc_an.txt
