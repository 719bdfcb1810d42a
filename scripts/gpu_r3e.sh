#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "min_chunk=2" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given --probes 0 "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "min_chunk=4" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --reps 4 --out gpurun_out/r3e_route.json > gpurun_out/r3e_route.log 2>&1; tail -1 gpurun_out/r3e_route.log
