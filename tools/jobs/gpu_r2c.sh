#!/bin/bash
# Reference anchors for C4's right-hand sides 1-7 and the apply_* anchors on
# the GPU-box host (reference from the git-ignored install baseline/_ref),
# in parallel with the GPU tests and the reference's own tests through the
# drop-in alias; then (host idle again) C3 sweep layout timings and the C4
# bench line.
mkdir -p gpurun_out/anchors
O=gpurun_out
export HELMSWEEP_REF=$PWD/baseline/_ref OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1
pids=""
for r in 1 2 3 4 5 6 7; do
  python tests/golden/make_large_anchors.py --out=$O/anchors/c4_r$r.json C4_rhs$r > $O/anchors/c4_r$r.log 2>&1 &
  pids="$pids $!"
done
python tests/golden/make_large_anchors.py --out=$O/anchors/apply_c4.json apply_C4 > $O/anchors/apply_c4.log 2>&1 &
pids="$pids $!"
(python tests/golden/make_large_anchors.py --out=$O/anchors/apply_c12.json apply_C2 apply_C1 > $O/anchors/apply_c12.log 2>&1) &
pids="$pids $!"
unset OMP_NUM_THREADS OPENBLAS_NUM_THREADS
timeout 900 python -m pytest tests -q -m gpu > $O/gputest3.log 2>&1; echo "gputest rc=$?" >> $O/rc3.txt
timeout 1200 bash tools/run_reference_tests.sh run -q --durations=15 > $O/reftests2.log 2>&1; echo "reftests rc=$?" >> $O/rc3.txt
for p in $pids; do wait $p; done
echo "anchors done" >> $O/rc3.txt
for cg in "16 0" "8 8" "16 3" "11 6" "12 6"; do
  set -- $cg
  HS_SWEEP_CPC=$1 HS_SWEEP_SEGMENTS=$2 timeout 300 python tools/time_sweep.py 2 >> $O/sweep_layouts.log 2>&1
  echo "C=$1 G=$2 rc=$?" >> $O/sweep_layouts.log
done
timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4.log 2>&1; echo "c4 rc=$?" >> $O/rc3.txt
echo done >> $O/rc3.txt
