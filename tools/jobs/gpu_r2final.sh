#!/bin/bash
# Round-2 final measurement set (one B200): GPU tests, bench lines of every
# config, the reference arm, launch list and ncu captures.  Every ncu command
# runs after the same command exited 0 without ncu.
mkdir -p gpurun_out
O=gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $O/host_fin.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/gputest_fin.log 2>&1; echo "gputest rc=$?" >> $O/rc_fin.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_fin.log 2>&1; echo "smoke rc=$?" >> $O/rc_fin.txt
timeout 900 python bench.py > $O/bench_c3_fin.log 2>&1; echo "c3 rc=$?" >> $O/rc_fin.txt
timeout 900 python bench.py --impl reference > $O/bench_ref_fin.log 2>&1; echo "ref rc=$?" >> $O/rc_fin.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_fin.log 2>&1; echo "c2 rc=$?" >> $O/rc_fin.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_fin.log 2>&1; echo "c4 rc=$?" >> $O/rc_fin.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_fin.log 2>&1; echo "c5 rc=$?" >> $O/rc_fin.txt
timeout 1200 python tools/time_many.py 4 1 1 2 4 > $O/many_c5_fin.log 2>&1; echo "many c5 rc=$?" >> $O/rc_fin.txt
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 600 $B > $O/plain_fin.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches_c3_fin.csv $B > $O/ncu_launch_fin.log 2>&1; echo "launch rc=$?" >> $O/rc_fin.txt
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_part_solve -c 3 -o $O/prof_sweep_c3_fin -f $B > $O/ncu_full_fin.log 2>&1; echo "ncu c3 rc=$?" >> $O/rc_fin.txt
timeout 600 python tools/time_many.py 3 1 4 > $O/many_c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_part_solve -s 33 -c 3 \
    -o $O/prof_sweep_c4_nr4 -f python tools/time_many.py 3 1 4 > $O/ncu_nr4_fin.log 2>&1; echo "ncu nr4 rc=$?" >> $O/rc_fin.txt
echo done >> $O/rc_fin.txt
timeout 1200 bash tools/run_reference_tests.sh run > $O/reftests_fin.log 2>&1; echo "reftests rc=$?" >> $O/rc_fin.txt
echo done2 >> $O/rc_fin.txt
