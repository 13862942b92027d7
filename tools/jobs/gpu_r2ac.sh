#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "many or lanes" > $O/many_tests2.log 2>&1; echo "tests rc=$?" >> $O/rc_ac.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --batch > $O/bench_c4_batch2.log 2>&1; echo "c4 batch g2 rc=$?" >> $O/rc_ac.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --batch --batch-groups 1 > $O/bench_c4_batch1.log 2>&1; echo "c4 batch g1 rc=$?" >> $O/rc_ac.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --batch --batch-groups 4 --segments 1 > $O/bench_c4_batch4.log 2>&1; echo "c4 batch g4 rc=$?" >> $O/rc_ac.txt
echo done >> $O/rc_ac.txt
