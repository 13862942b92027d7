#!/bin/bash
# C5 full-size reference anchor on the GPU-box host (needs ~60-80 GB of host
# RAM, which the build container does not have), alongside an ncu traffic
# capture of one whole C3 X application (3 k_part_solve launches).
mkdir -p gpurun_out/anchors
O=gpurun_out
(HELMSWEEP_REF=$PWD/baseline/_ref OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 timeout 3200 \
  python tests/golden/make_large_anchors.py --out=$O/anchors/c5.json C5 apply_C5 > $O/anchors/c5.log 2>&1; \
  echo "c5 anchor rc=$?" >> $O/rc8.txt) &
apid=$!
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_part_solve -c 3 -o $O/prof_sweep_c3_app -f $B > $O/ncu_full2.log 2>&1; echo "ncu rc=$?" >> $O/rc8.txt
timeout 600 python -m pytest tests/test_line1d.py -q -m gpu > $O/gputest8.log 2>&1; echo "gputest rc=$?" >> $O/rc8.txt
while kill -0 $apid 2>/dev/null; do sleep 20; free -g | sed -n 2p >> $O/anchors/c5_mem.log; done
echo done >> $O/rc8.txt
