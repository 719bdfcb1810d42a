#!/bin/bash
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_c3.py tests/test_gpu_parity.py tests/test_gpu_stream.py 2>&1 | tail -3
timeout 600 python scripts/sweep_opts.py "" "min_chunk=3" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --out gpurun_out/r4j_route.json > gpurun_out/r4j_a.log 2>&1; tail -c 400 gpurun_out/r4j_a.log
