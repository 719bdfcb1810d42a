#!/bin/bash
timeout 300 python scripts/trace_step.py --out gpurun_out/r4d_route.json > gpurun_out/r4d_route.log 2>&1; tail -c 300 gpurun_out/r4d_route.log
timeout 300 python scripts/trace_step.py --opt min_chunk=3 --opt fetch_lead=1 --out gpurun_out/r4d_route3.json > gpurun_out/r4d_route3.log 2>&1; tail -c 300 gpurun_out/r4d_route3.log
