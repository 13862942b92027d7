#!/bin/bash
# C4 lockstep batches: more cluster layouts for two groups
mkdir -p gpurun_out
O=gpurun_out
run() {
  label=$1; shift
  env "$@" timeout 900 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline $EXTRA 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],1), d['iterations'], d.get('sweep_segments'), d.get('rhs_per_chain'), d.get('rhs_mode')[:22])" >> $O/c4_layouts2.log
}
EXTRA="--segments 5" run "groups2_C6_G5" HS_SWEEP_CPC=6
EXTRA="--segments 4" run "groups2_C8_G4" HS_SWEEP_CPC=8
EXTRA="--segments 8" run "groups2_C4_G8" HS_SWEEP_CPC=4
EXTRA="--segments 6" run "groups2_C5_G6" HS_SWEEP_CPC=5
EXTRA="--segments 4" run "groups2_C6_G4" HS_SWEEP_CPC=6
EXTRA="--segments 3" run "groups2_C8_G3" HS_SWEEP_CPC=8
echo done >> $O/c4_layouts2.log
