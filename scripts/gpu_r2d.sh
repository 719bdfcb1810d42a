#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --out gpurun_out/r2d_trace.json > gpurun_out/r2d_trace.log 2>&1; tail -5 gpurun_out/r2d_trace.log
timeout 600 python scripts/trace_step.py --opt decode_wait=1 --out gpurun_out/r2d_trace_wait.json > gpurun_out/r2d_trace_wait.log 2>&1; tail -3 gpurun_out/r2d_trace_wait.log
