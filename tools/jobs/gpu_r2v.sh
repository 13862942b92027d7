#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest18.log 2>&1; echo "gputest rc=$?" >> $O/rc18.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3_z.log 2>&1; echo "c3 rc=$?" >> $O/rc18.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_z.log 2>&1; echo "c2 rc=$?" >> $O/rc18.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_z.log 2>&1; echo "c4 rc=$?" >> $O/rc18.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_z.log 2>&1; echo "c5 rc=$?" >> $O/rc18.txt
echo done >> $O/rc18.txt
