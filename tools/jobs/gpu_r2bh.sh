#!/bin/bash
# C4 lockstep batches: four groups of two
mkdir -p gpurun_out
O=gpurun_out
run() {
  label=$1; shift
  env "$@" timeout 900 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline $EXTRA 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],1), d['iterations'], d.get('sweep_segments'), d.get('rhs_per_chain'), d.get('rhs_mode')[:22])" >> $O/c4_layouts3.log
}
EXTRA="--batch-groups 4 --segments 2" run "groups4_C6_G2" HS_SWEEP_CPC=6
EXTRA="--batch-groups 4 --segments 3" run "groups4_C5_G3" HS_SWEEP_CPC=5
EXTRA="--batch-groups 4 --segments 2" run "groups4_C8_G2" HS_SWEEP_CPC=8
EXTRA="--batch-groups 4 --segments 2" run "groups4_C9_G1x" HS_SWEEP_CPC=9
EXTRA="--batch-groups 3 --segments 3" run "groups3_C6_G3" HS_SWEEP_CPC=6
echo done >> $O/c4_layouts3.log
