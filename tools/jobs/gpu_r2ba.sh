#!/bin/bash
# ncu --set full of the 3-D kernels with 4 right-hand sides per chain (C5 coarse level)
mkdir -p gpurun_out
O=gpurun_out
export HS_MANY_ONLY=1
timeout 900 python tools/time_many.py 4 1 4 > $O/many_c5_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k3_solve|k3_gemv" -s 8 -c 4 \
   -o $O/prof_3d_nr4 -f python tools/time_many.py 4 1 4 > $O/ncu_3d_nr4.log 2>&1; echo "ncu rc=$?" > $O/rc_ba.txt
