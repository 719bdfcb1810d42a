#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "chunk=4" "chunk=16" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --given --reps 4 --out gpurun_out/r2t_given.json > gpurun_out/r2t_given.log 2>&1; tail -1 gpurun_out/r2t_given.log
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_c3.py tests/test_gpu_regressions.py tests/test_gpu_append.py -q -x --timeout 400 -p no:cacheprovider 2>&1 | tail -3
