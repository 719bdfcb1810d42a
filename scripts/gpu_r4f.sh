#!/bin/bash
timeout 300 python scripts/trace_step.py --given --opt debug_skip=2 --out gpurun_out/r4f_given_skip2.json > gpurun_out/r4f_a.log 2>&1; tail -c 300 gpurun_out/r4f_a.log
timeout 300 python scripts/trace_step.py --given --out gpurun_out/r4f_given.json > gpurun_out/r4f_b.log 2>&1; tail -c 300 gpurun_out/r4f_b.log
timeout 300 python scripts/trace_step.py --opt debug_skip=2 --out gpurun_out/r4f_route_skip2.json > gpurun_out/r4f_c.log 2>&1; tail -c 300 gpurun_out/r4f_c.log
