#!/bin/bash
# level-0 sparse couplings streamed through the ring (HS_SWEEP_CPL0=1) vs the default alpha / gamma blocks
mkdir -p gpurun_out
O=gpurun_out
HS_SWEEP_CPL0=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sweeps or tgsp_apply or many or C2" > $O/cpl_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_aq.txt
for k in 1 2; do
for cfg in 2 1 3; do
  echo -n "default: " >> $O/cpl_ring_ab.log; python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/cpl_ring_ab.log
  echo -n "cpl0=1 : " >> $O/cpl_ring_ab.log; HS_SWEEP_CPL0=1 python tools/time_sweep.py $cfg 2>&1 | tail -n 1 | cut -c20- >> $O/cpl_ring_ab.log
done
done
echo "default:" >> $O/cpl_ring_ab.log; python tools/time_many.py 3 1 4 2>&1 | grep "x:" >> $O/cpl_ring_ab.log
echo "cpl0=1:" >> $O/cpl_ring_ab.log; HS_SWEEP_CPL0=1 python tools/time_many.py 3 1 4 2>&1 | grep "x:" >> $O/cpl_ring_ab.log
echo done >> $O/rc_aq.txt
