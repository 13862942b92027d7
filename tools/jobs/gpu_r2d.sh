#!/bin/bash
# GPU tests, the reference's tests through the alias, C5 sweep timing and bench line
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -q -m gpu > $O/gputest4.log 2>&1; echo "gputest rc=$?" >> $O/rc4.txt
timeout 1200 bash tools/run_reference_tests.sh run -q --durations=20 > $O/reftests3.log 2>&1; echo "reftests rc=$?" >> $O/rc4.txt
timeout 600 python tools/time_sweep3.py > $O/sweep3.log 2>&1; echo "sweep3 rc=$?" >> $O/rc4.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "c5 rc=$?" >> $O/rc4.txt
echo done >> $O/rc4.txt
