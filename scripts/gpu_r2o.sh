#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --given --reps 4 --out gpurun_out/r2o_given.json > gpurun_out/r2o_given.log 2>&1; tail -1 gpurun_out/r2o_given.log
timeout 300 python scripts/sweep_opts.py "" "chunk=4" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" 2>&1 | tail -1
