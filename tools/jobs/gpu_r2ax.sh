#!/bin/bash
mkdir -p gpurun_out
for cfg in 1 2 4; do timeout 900 python tools/gate_stats.py $cfg >> gpurun_out/gate_stats.log 2>&1; done
echo done >> gpurun_out/gate_stats.log
