#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -x -m gpu -k "3d or exact or factorize or line1d or C5 or deterministic or stencil27" > $O/tests3d.log 2>&1; echo "tests3d rc=$?" >> $O/rc_ai.txt
timeout 900 python tools/time_sweep3.py > $O/sweep3_new.log 2>&1
HS_LIB=variants/libold.so timeout 900 python tools/time_sweep3.py > $O/sweep3_old.log 2>&1
echo done >> $O/rc_ai.txt
