#!/bin/bash
# 3-D chains: both fronts' chains interleaved on every CTA (default) vs split CTA groups (HS_S3_SPLIT=1)
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -x -m gpu -k "3d or exact or factorize or line1d or C5 or deterministic or many" > $O/tests3d_at.log 2>&1; echo "tests3d rc=$?" >> $O/rc_at.txt
for k in 1 2; do
  echo -n "interleaved: " >> $O/s3_inter_ab.log; timeout 900 python tools/time_sweep3.py 2>&1 | tail -n 1 >> $O/s3_inter_ab.log
  echo -n "split      : " >> $O/s3_inter_ab.log; HS_S3_SPLIT=1 timeout 900 python tools/time_sweep3.py 2>&1 | tail -n 1 >> $O/s3_inter_ab.log
done
timeout 900 python tools/time_many.py 4 1 1 2 4 > $O/many_c5_inter.log 2>&1
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_inter.log 2>&1; echo "c5 rc=$?" >> $O/rc_at.txt
echo done >> $O/rc_at.txt
