#!/bin/bash
# sharded path after z-keeping: GPU shard tests, logical-shard bench at C2, new argument-error test
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_shards.py tests/test_gpu_parity.py -q -x -m gpu -k "shard or argument_errors" > $O/shard_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_ap.txt
for g in 1 2 4; do
  timeout 600 python bench.py --config 1 --shard --local-shards $g --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c2_shard$g.log 2>&1; echo "shard $g rc=$?" >> $O/rc_ap.txt
done
echo done >> $O/rc_ap.txt
