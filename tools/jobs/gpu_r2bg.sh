#!/bin/bash
# cluster option: test, C4 default bench line (two batches on 6-CTA clusters), full GPU tests
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_option or c4_lockstep" > $O/cluster_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_bg.txt
timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_c4_bg.log 2>&1; echo "c4 rc=$?" >> $O/rc_bg.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_bg.log 2>&1; echo "gputest rc=$?" >> $O/rc_bg.txt
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > $O/bench_c3_bg.log 2>&1; echo "c3 rc=$?" >> $O/rc_bg.txt
echo done >> $O/rc_bg.txt
