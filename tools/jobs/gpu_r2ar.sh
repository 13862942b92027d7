#!/bin/bash
# forward levels: longest-processing-time warp assignment (default) vs round-robin (variants/librr.so)
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sweeps or tgsp_apply or many or C2 or nx or subdom or determin" > $O/lpt_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_ar.txt
for k in 1 2; do
for cfg in 2 1 3; do
  echo -n "lpt: " >> $O/lpt_ab.log; python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/lpt_ab.log
  echo -n "rr : " >> $O/lpt_ab.log; HS_LIB=variants/librr.so python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/lpt_ab.log
done
done
echo "lpt:" >> $O/lpt_ab.log; python tools/time_many.py 3 1 2 4 2>&1 | grep "x:" >> $O/lpt_ab.log
echo "rr:" >> $O/lpt_ab.log; HS_LIB=variants/librr.so python tools/time_many.py 3 1 2 4 2>&1 | grep "x:" >> $O/lpt_ab.log
echo done >> $O/rc_ar.txt
