#!/bin/bash
# time_sweep.py for the default library and every variants/*.so (A/B experiments)
cfg=${1:-1}
python tools/time_sweep.py $cfg
for v in variants/*.so; do
  [ -e "$v" ] || continue
  echo -n "$v: "; HS_LIB=$v python tools/time_sweep.py $cfg
done
