#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --given --reps 6 --out gpurun_out/r2l_given.json > gpurun_out/r2l_given.log 2>&1; tail -1 gpurun_out/r2l_given.log
timeout 600 python scripts/trace_step.py --reps 6 --out gpurun_out/r2l_route.json > gpurun_out/r2l_route.log 2>&1; tail -1 gpurun_out/r2l_route.log
timeout 600 python scripts/trace_step.py --dense --reps 4 --out gpurun_out/r2l_dense.json > gpurun_out/r2l_dense.log 2>&1; tail -1 gpurun_out/r2l_dense.log
