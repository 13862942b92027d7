#!/bin/bash
# Round profile: bench line, launch list of one timed GMRES solve, and one
# ncu --set full capture of the sweep kernel (run under gpurun, 1 GPU).
set -e
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
T="python tools/time_sweep.py 1"
$B > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-3600} -c ${COUNT:-1100} \
    --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
$T > gpurun_out/plain_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_part_solve -s 8 -c 4 \
    -o gpurun_out/prof -f $T > gpurun_out/ncu_full.log 2>&1
echo done
