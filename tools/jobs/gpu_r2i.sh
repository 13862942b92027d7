#!/bin/bash
# level-0 sparse couplings A/B (HS_SWEEP_CPL0=0: streamed alpha/gamma blocks)
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > $O/gputest9.log 2>&1; echo "gputest rc=$?" >> $O/rc9.txt
for cfg in 1 2 3; do
  HS_SWEEP_CPL0=0 timeout 300 python tools/time_sweep.py $cfg >> $O/cpl0_ab.log 2>&1
  timeout 300 python tools/time_sweep.py $cfg >> $O/cpl0_ab.log 2>&1
done
echo "ab rc=$?" >> $O/rc9.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3_cpl0.log 2>&1; echo "bench rc=$?" >> $O/rc9.txt
echo done >> $O/rc9.txt
