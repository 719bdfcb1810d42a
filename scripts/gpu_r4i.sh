#!/bin/bash
timeout 600 python scripts/sweep_opts.py "" "decode_wait=1" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --opt decode_wait=1 --out gpurun_out/r4i_wait.json > gpurun_out/r4i_a.log 2>&1; tail -c 1500 gpurun_out/r4i_a.log
