#!/bin/bash
# what the driver runs at round end, on HEAD: GPU tests, smoke(), the default bench line, the reference arm
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/last_gputest.log 2>&1; echo "gputest rc=$?" >> $O/rc_last.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/last_smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc_last.txt
timeout 900 python bench.py > $O/last_bench.log 2>&1; echo "bench rc=$?" >> $O/rc_last.txt
timeout 900 python bench.py --impl reference > $O/last_ref.log 2>&1; echo "ref rc=$?" >> $O/rc_last.txt
echo done >> $O/rc_last.txt
