#!/bin/bash
timeout 300 python scripts/trace_step.py --reps 4 --out gpurun_out/r4k_route.json > gpurun_out/r4k_a.log 2>&1; tail -c 300 gpurun_out/r4k_a.log
