#!/bin/bash
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_stream.py tests/test_gpu_c3.py 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --reps 6 --out gpurun_out/r4z_route.json > gpurun_out/r4z_a.log 2>&1; tail -c 100 gpurun_out/r4z_a.log
