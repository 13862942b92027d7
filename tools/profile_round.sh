#!/bin/bash
# Round profile (run under gpurun, 1 GPU): bench lines of every BASELINE
# config, the reference arm, the launch list of one timed C2 GMRES solve, and
# ncu --set full captures of the 2-D sweep kernel (C2), the fine stencil
# kernels (C2) and the 3-D chain kernel (C5).  Every ncu command runs only
# after the same command exited 0 without ncu.
set -e
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
T="python tools/time_sweep.py 1"
S="python tools/time_stencil.py 1"
python bench.py > gpurun_out/bench_c2_full.log 2>&1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
$B > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-3400} -c ${COUNT:-1100} \
    --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
$T > gpurun_out/plain_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_part_solve -s 8 -c 4 \
    -o gpurun_out/prof -f $T > gpurun_out/ncu_full.log 2>&1
$S > gpurun_out/plain_stencil.log 2>&1
ncu --set full --clock-control none -k regex:k_stencil -s 20 -c 8 \
    -o gpurun_out/prof_stencil -f $S > gpurun_out/ncu_stencil.log 2>&1
ncu --set full --clock-control none -k regex:"k_pre2d|k_post2d" -s 10 -c 2 \
    -o gpurun_out/prof_fused -f $B > gpurun_out/ncu_fused.log 2>&1
echo done
