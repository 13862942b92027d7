#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_c4_bj.log 2>&1; echo "c4 rc=$?" >> $O/rc_bj.txt
timeout 900 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline --batch-groups 2 > $O/bench_c4_bj2.log 2>&1; echo "c4 g2 rc=$?" >> $O/rc_bj.txt
echo done >> $O/rc_bj.txt
