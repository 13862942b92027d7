#!/bin/bash
# C4 lockstep batches: cluster layouts for two groups
mkdir -p gpurun_out
O=gpurun_out
run() { # label, env..., args
  label=$1; shift
  env "$@" timeout 900 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline $EXTRA 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],1), d['iterations'], d.get('sweep_segments'), d.get('rhs_per_chain'))" >> $O/c4_layouts.log
}
EXTRA="" run "groups2_C9_G3" X=1
EXTRA="--batch-groups 1" run "groups1_C9_G7" X=1
EXTRA="--segments 6" run "groups2_C6_G6" HS_SWEEP_CPC=6
EXTRA="--segments 4" run "groups2_C7_G4" HS_SWEEP_CPC=7
EXTRA="--segments 5" run "groups2_C6_G5" HS_SWEEP_CPC=6
echo done >> $O/c4_layouts.log
