#!/bin/bash
# GPU tests (full), the reference's own hot-path tests through the drop-in
# alias, C5 bench line and C4 multi-RHS layouts.
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu > $O/gputest2.log 2>&1; echo "gputest rc=$?" >> $O/rc2.txt
timeout 1200 bash tools/run_reference_tests.sh run -x -q --durations=15 > $O/reftests.log 2>&1; echo "reftests rc=$?" >> $O/rc2.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "c5 rc=$?" >> $O/rc2.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --lanes 1 > $O/bench_c4_l1.log 2>&1; echo "c4 l1 rc=$?" >> $O/rc2.txt
HS_SWEEP_SEGMENTS=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --lanes 4 > $O/bench_c4_g1l4.log 2>&1; echo "c4 g1 l4 rc=$?" >> $O/rc2.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --lanes 2 > $O/bench_c4_l2.log 2>&1; echo "c4 l2 rc=$?" >> $O/rc2.txt
echo done >> $O/rc2.txt
