#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out
for cpc in 9 12; do
  for lanes in 4 6 7 8; do
    r=$(HS_SWEEP_CPC=$cpc timeout 400 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline \
        --lanes $lanes --segments 1 --clock-sampler none 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null)
    echo "cpc=$cpc lanes=$lanes ms=$r" >> $O/c4_layouts2.log
  done
done
echo done >> $O/c4_layouts2.log
