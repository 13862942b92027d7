#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/profile_batch.py 3 > gpurun_out/profile_batch_c4.log 2>&1; echo "rc=$?" >> gpurun_out/profile_batch_c4.log
