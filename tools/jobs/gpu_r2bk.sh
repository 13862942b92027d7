#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c4_lockstep or batches_on_lanes or cluster_option" > gpurun_out/c4_batch_test2.log 2>&1; echo "rc=$?" >> gpurun_out/c4_batch_test2.log
