#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --given --reps 4 --out gpurun_out/r2s_given.json > gpurun_out/r2s_given.log 2>&1; tail -1 gpurun_out/r2s_given.log
timeout 300 python scripts/trace_step.py --given --opt debug_skip=1 --reps 4 --out gpurun_out/r2s_skip.json > gpurun_out/r2s_skip.log 2>&1; tail -1 gpurun_out/r2s_skip.log
