#!/bin/bash
# re-orthogonalisation threshold eta = 0.1 (Rutishauser) vs 1/sqrt(2) (DGKS): parity tests and solve times
mkdir -p gpurun_out
O=gpurun_out
export HS_DGKS_ETA=0.1
timeout 1500 python -m pytest tests -q -m gpu > $O/eta_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_ay.txt
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > $O/bench_c3_eta.log 2>&1; echo "c3 rc=$?" >> $O/rc_ay.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_eta.log 2>&1; echo "c2 rc=$?" >> $O/rc_ay.txt
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_c4_eta.log 2>&1; echo "c4 rc=$?" >> $O/rc_ay.txt
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_eta.log 2>&1; echo "c5 rc=$?" >> $O/rc_ay.txt
echo done >> $O/rc_ay.txt
