#!/bin/bash
# round 2: C3 step timeline (trace) + option sweep
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --out gpurun_out/r2i_trace.json > gpurun_out/r2i_trace.log 2>&1; tail -3 gpurun_out/r2i_trace.log
timeout 600 python scripts/sweep_opts.py "" "chunk=4" "chunk=16" "decode_wait=1" "cluster_route=0" 2>&1 | tail -8
