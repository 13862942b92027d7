#!/bin/bash
# GPU tests, C5 setup + sweep timing and bench line after the hand-written 3-D factorisation
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > $O/gputest5.log 2>&1; echo "gputest rc=$?" >> $O/rc5.txt
timeout 900 python tools/time_sweep3.py > $O/sweep3b.log 2>&1; echo "sweep3 rc=$?" >> $O/rc5.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5b.log 2>&1; echo "c5 rc=$?" >> $O/rc5.txt
echo done >> $O/rc5.txt
