#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --batch > $O/bench_c4_batch.log 2>&1; echo "c4 batch rc=$?" >> $O/rc_ab.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_lanes.log 2>&1; echo "c4 lanes rc=$?" >> $O/rc_ab.txt
echo done >> $O/rc_ab.txt
