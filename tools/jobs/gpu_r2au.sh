#!/bin/bash
# reference tests through the alias at HEAD (multi-column Factorization.solve is now one batched solve) + new test
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gmres_many" > $O/gm3d_tests.log 2>&1; echo "tests rc=$?" >> $O/rc_au.txt
timeout 1200 bash tools/run_reference_tests.sh run > $O/reftests_au.log 2>&1; echo "reftests rc=$?" >> $O/rc_au.txt
echo done >> $O/rc_au.txt
