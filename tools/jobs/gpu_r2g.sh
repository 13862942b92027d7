#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest7.log 2>&1; echo "gputest rc=$?" >> $O/rc7.txt
timeout 600 python tools/time_relay.py 2 1 2 4 8 > $O/relay_c3.json 2>$O/relay_c3.err; echo "relay c3 rc=$?" >> $O/rc7.txt
timeout 600 python tools/time_relay.py 1 1 2 4 8 > $O/relay_c2.json 2>$O/relay_c2.err; echo "relay c2 rc=$?" >> $O/rc7.txt
timeout 900 python bench.py > $O/bench_c3_r2.log 2>&1; echo "bench rc=$?" >> $O/rc7.txt
timeout 900 python bench.py --impl reference > $O/bench_ref_r2.log 2>&1; echo "ref rc=$?" >> $O/rc7.txt
echo done >> $O/rc7.txt
