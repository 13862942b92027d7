#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest16.log 2>&1; echo "gputest rc=$?" >> $O/rc16.txt
timeout 900 python bench.py > $O/bench_c3_final.log 2>&1; echo "c3 rc=$?" >> $O/rc16.txt
timeout 900 python bench.py --impl reference > $O/bench_ref_final.log 2>&1; echo "ref rc=$?" >> $O/rc16.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_final.log 2>&1; echo "c2 rc=$?" >> $O/rc16.txt
timeout 600 python tools/time_relay.py 2 1 2 4 8 > $O/relay_c3_final.json 2>/dev/null; echo "relay rc=$?" >> $O/rc16.txt
echo done >> $O/rc16.txt
