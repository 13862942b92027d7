#!/bin/bash
# first-pass update fused with the second pass's dots (default) vs the plain update kernel (the second pass rarely runs now)
mkdir -p gpurun_out
O=gpurun_out
for k in 1 2; do
  timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fused   c3', d['ms_per_step'], d['iterations'])" >> $O/update_ab.log
  HS_FUSE_UPDATE_DOT=0 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('unfused c3', d['ms_per_step'], d['iterations'])" >> $O/update_ab.log
done
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fused   c2', d['ms_per_step'], d['iterations'])" >> $O/update_ab.log
HS_FUSE_UPDATE_DOT=0 timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('unfused c2', d['ms_per_step'], d['iterations'])" >> $O/update_ab.log
echo done >> $O/update_ab.log
