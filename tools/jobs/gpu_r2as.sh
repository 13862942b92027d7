#!/bin/bash
# soak: the threaded multi-right-hand-side paths 15 times over (flakiness check)
mkdir -p gpurun_out
O=gpurun_out
pass=0; fail=0
for i in $(seq 1 15); do
  if timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "batches_on_lanes or lanes_match or gmres_many" > $O/soak_$i.log 2>&1; then pass=$((pass+1)); else fail=$((fail+1)); cp $O/soak_$i.log $O/soak_fail_$i.log; fi
done
echo "pass=$pass fail=$fail" > $O/soak.txt
timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_c4_soak.log 2>&1; echo "c4 rc=$?" >> $O/soak.txt
