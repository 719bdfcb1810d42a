#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --given --reps 4 --out gpurun_out/r2p_given.json > gpurun_out/r2p_given.log 2>&1; tail -1 gpurun_out/r2p_given.log
timeout 300 python scripts/trace_step.py --given --opt debug_skip=1 --reps 4 --out gpurun_out/r2p_given_skip.json > gpurun_out/r2p_given_skip.log 2>&1; tail -1 gpurun_out/r2p_given_skip.log
timeout 300 python scripts/sweep_opts.py "" "debug_skip=1" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "debug_skip=1" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ref_suite.py -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
