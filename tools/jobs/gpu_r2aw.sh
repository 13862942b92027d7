#!/bin/bash
# k_post2d with the prolongation operands staged in shared memory: bitwise tests, timing vs the previous library
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or tgsp or C2 or C3 or C4 or gmres_iter or transfers" > $O/post_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_aw.txt
for cfg in 2 1 3; do
  echo "new:" >> $O/post_ab.log; python tools/time_fused.py $cfg 2>&1 | grep fused >> $O/post_ab.log
  echo "old:" >> $O/post_ab.log; HS_LIB=variants/libprev.so python tools/time_fused.py $cfg 2>&1 | grep fused >> $O/post_ab.log
done
echo done >> $O/rc_aw.txt
