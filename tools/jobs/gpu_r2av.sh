#!/bin/bash
# ncu --set full of the fine-level and Krylov kernels inside one timed C3 solve
mkdir -p gpurun_out
O=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --clock-sampler none"
timeout 600 $B > $O/plain_av.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_pre2d|k_post2d|k_stencil|k_block|k_restrict|k_scale_inv" -s 40 -c 16 -o $O/prof_fine_c3 -f $B > $O/ncu_fine.log 2>&1; echo "ncu fine rc=$?" > $O/rc_av.txt
