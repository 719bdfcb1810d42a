#!/bin/bash
timeout 300 python scripts/trace_step.py --given --opt debug_skip=1 --out gpurun_out/r4g_given_skip1.json > gpurun_out/r4g_a.log 2>&1; tail -c 200 gpurun_out/r4g_a.log
timeout 300 python scripts/trace_step.py --opt debug_skip=1 --out gpurun_out/r4g_route_skip1.json > gpurun_out/r4g_c.log 2>&1; tail -c 200 gpurun_out/r4g_c.log
