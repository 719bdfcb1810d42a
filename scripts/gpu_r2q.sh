#!/bin/bash
# ncu source-level capture of the decode kernel (given lists: no routing kernel alongside)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 4 -c 1 \
    -o gpurun_out/r2q_decode python scripts/trace_step.py --plain --given --reps 6 > gpurun_out/r2q_ncu.log 2>&1; tail -3 gpurun_out/r2q_ncu.log
timeout 900 python -m pytest tests/test_gpu_ref_suite.py tests/test_gpu_comm.py -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
