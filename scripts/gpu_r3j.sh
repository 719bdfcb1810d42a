#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --reps 4 --out gpurun_out/r3j_route.json > gpurun_out/r3j_route.log 2>&1; tail -1 gpurun_out/r3j_route.log
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_c3.py tests/test_gpu_append.py -q -x --timeout 400 -p no:cacheprovider 2>&1 | tail -2
