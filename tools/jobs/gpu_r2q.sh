#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest17.log 2>&1; echo "gputest rc=$?" >> $O/rc17.txt
timeout 600 python tools/time_relay.py 1 1 2 4 8 > $O/relay_c2_final.json 2>/dev/null
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_final.log 2>&1; echo "c4 rc=$?" >> $O/rc17.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_final.log 2>&1; echo "c5 rc=$?" >> $O/rc17.txt
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches_c3_final.csv $B > $O/ncu_launch2.log 2>&1; echo "launch rc=$?" >> $O/rc17.txt
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_part_solve -c 3 -o $O/prof_sweep_c3_c9 -f $B > $O/ncu_full3.log 2>&1; echo "ncu rc=$?" >> $O/rc17.txt
echo done >> $O/rc17.txt
