#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --reps 4 --out gpurun_out/r2w_route.json > gpurun_out/r2w_route.log 2>&1; tail -1 gpurun_out/r2w_route.log
timeout 300 python scripts/sweep_opts.py "" "chunk=6" 2>&1 | tail -1
