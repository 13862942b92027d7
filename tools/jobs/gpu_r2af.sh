#!/bin/bash
# (1) NR = 1 kernel before/after the multi-right-hand-side change (same box)
# (2) full GPU test suite (3) ncu of one NR = 4 application at C4
mkdir -p gpurun_out
O=gpurun_out
for k in 1 2; do
  for cfg in 2 1 3; do
    python tools/time_sweep.py $cfg >> $O/ab_new.log 2>&1
    HS_LIB=variants/libold.so python tools/time_sweep.py $cfg >> $O/ab_old.log 2>&1
  done
done
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_af.log 2>&1; echo "gputest rc=$?" >> $O/rc_af.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_part_solve -s 12 -c 3 \
   -o $O/prof_sweep_c4_nr4 -f python tools/time_many.py 3 1 4 > $O/ncu_nr4.log 2>&1; echo "ncu rc=$?" >> $O/rc_af.txt
echo done >> $O/rc_af.txt
