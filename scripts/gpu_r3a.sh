#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --dense --ctx-len 8192 --reps 4 --out gpurun_out/r3a_dense8k.json > gpurun_out/r3a_dense8k.log 2>&1; tail -1 gpurun_out/r3a_dense8k.log
timeout 300 python scripts/trace_step.py --given --probes 0 --reps 4 --out gpurun_out/r3a_win.json > gpurun_out/r3a_win.log 2>&1; tail -1 gpurun_out/r3a_win.log
