#!/bin/bash
# Round-2 GPU pass (gpurun, 1 GPU): GPU tests, the default bench line (C3,
# with the CPU baseline), the reference arm, bench lines of C2/C4/C5, the
# launch list of one timed C3 solve (bench's timed region only, via
# cudaProfilerStart/Stop) and an ncu --set full capture of the 2-D slab-solve
# kernel at C3.  Every ncu command runs after the same command exited 0
# without ncu.
mkdir -p gpurun_out
O=gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $O/host.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_c3.log 2>&1; echo "bench c3 rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/rc.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2.log 2>&1; echo "c2 rc=$?" >> $O/rc.txt
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4.log 2>&1; echo "c4 rc=$?" >> $O/rc.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "c5 rc=$?" >> $O/rc.txt
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 600 $B > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches_c3.csv $B > $O/ncu_launch.log 2>&1; echo "launch rc=$?" >> $O/rc.txt
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_part_solve -c 2 -o $O/prof_sweep_c3 -f $B > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/rc.txt
echo done >> $O/rc.txt
