#!/bin/bash
# round 2: full C3 bench with parity + step traces
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; tail -c 5000 gpurun_out/r2c_bench.json; tail -5 gpurun_out/r2c_bench.err
timeout 600 python scripts/trace_step.py --out gpurun_out/r2c_trace.json > gpurun_out/r2c_trace.log 2>&1; tail -5 gpurun_out/r2c_trace.log
