#!/bin/bash
# final round-2 measurement set (after the z-keeping GMRES)
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest_final.log 2>&1; echo "gputest rc=$?" >> $O/rc_final.txt
timeout 900 python bench.py > $O/bench_c3_fin.log 2>&1; echo "c3 rc=$?" >> $O/rc_final.txt
timeout 900 python bench.py --impl reference > $O/bench_ref_fin.log 2>&1; echo "ref rc=$?" >> $O/rc_final.txt
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 600 $B > $O/plain_fin.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches_c3_fin.csv $B > $O/ncu_launch_fin.log 2>&1; echo "launch rc=$?" >> $O/rc_final.txt
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_pre2d|k_post2d|k_stencil|k_block" -c 12 -o $O/prof_fine_c3 -f $B > $O/ncu_fine.log 2>&1; echo "ncu fine rc=$?" >> $O/rc_final.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_fin.log 2>&1; echo "smoke rc=$?" >> $O/rc_final.txt
echo done >> $O/rc_final.txt
