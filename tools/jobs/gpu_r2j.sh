#!/bin/bash
# C5: persistent two-task GEMV, sweep timing, bench line, ncu of the 3-D kernels
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "3d or pml3d or C5 or exact or factor or dense" > $O/gputest10.log 2>&1; echo "gputest rc=$?" >> $O/rc10.txt
timeout 900 python tools/time_sweep3.py > $O/sweep3c.log 2>&1; echo "sweep3 rc=$?" >> $O/rc10.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5c.log 2>&1; echo "c5 rc=$?" >> $O/rc10.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k3_solve|k3_gemv" -s 6 -c 4 \
   -o $O/prof_c5_3d -f python tools/time_sweep3.py > $O/ncu_c5.log 2>&1; echo "ncu rc=$?" >> $O/rc10.txt
echo done >> $O/rc10.txt
