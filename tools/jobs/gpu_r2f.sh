#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python -m pytest tests/test_line1d.py -q -m gpu > $O/gputest6.log 2>&1; echo "gputest rc=$?" >> $O/rc6.txt
timeout 600 python tools/time_relay.py 2 1 2 4 8 > $O/relay_c3.json 2>$O/relay_c3.err; echo "relay c3 rc=$?" >> $O/rc6.txt
timeout 600 python tools/time_relay.py 1 1 2 4 8 > $O/relay_c2.json 2>$O/relay_c2.err; echo "relay c2 rc=$?" >> $O/rc6.txt
echo done >> $O/rc6.txt
