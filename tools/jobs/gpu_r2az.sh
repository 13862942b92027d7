#!/bin/bash
# after the profiler-bytes change of the gated Krylov launches and the lane launch count: C4 and C3 lines, test pass
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_az.log 2>&1; echo "gputest rc=$?" >> $O/rc_az.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_az.log 2>&1; echo "c4 rc=$?" >> $O/rc_az.txt
timeout 900 python bench.py > $O/bench_c3_az.log 2>&1; echo "c3 rc=$?" >> $O/rc_az.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-batch > $O/bench_c4_lanes_az.log 2>&1; echo "c4 lanes rc=$?" >> $O/rc_az.txt
echo done >> $O/rc_az.txt
