#!/bin/bash
# new default layout (9-CTA clusters, co-resident segments): tests + bench lines
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest15.log 2>&1; echo "gputest rc=$?" >> $O/rc15.txt
for cfg in 0 1 2 3; do timeout 300 python tools/time_sweep.py $cfg >> $O/sweep_default.log 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3_l9.log 2>&1; echo "c3 rc=$?" >> $O/rc15.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_l9.log 2>&1; echo "c2 rc=$?" >> $O/rc15.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_l9.log 2>&1; echo "c4 rc=$?" >> $O/rc15.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --lanes 1 > $O/bench_c4_l9_seq.log 2>&1; echo "c4 seq rc=$?" >> $O/rc15.txt
timeout 600 python tools/time_nx.py > $O/nx_l9.log 2>&1; echo "nx rc=$?" >> $O/rc15.txt
echo done >> $O/rc15.txt
