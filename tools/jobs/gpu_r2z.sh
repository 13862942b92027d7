#!/bin/bash
# re-entry validation: GPU tests, default bench line, reference tests through the alias
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_z.log 2>&1; echo "gputest rc=$?" >> $O/rc_z.txt
timeout 900 python bench.py > $O/bench_c3_z.log 2>&1; echo "c3 rc=$?" >> $O/rc_z.txt
timeout 900 bash tools/run_reference_tests.sh run -q > $O/reftests_z.log 2>&1; echo "reftests rc=$?" >> $O/rc_z.txt
echo done >> $O/rc_z.txt
