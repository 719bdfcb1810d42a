#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "chunk=4" "chunk=6" "chunk=12" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "chunk_dense=8" "chunk_dense=32" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --reps 4 --out gpurun_out/r2u_route.json > gpurun_out/r2u_route.log 2>&1; tail -1 gpurun_out/r2u_route.log
