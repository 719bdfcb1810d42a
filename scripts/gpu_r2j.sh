#!/bin/bash
# round 2: routing exact path over DSMEM, one reserved ticket: trace + sweep + stream/parity tests
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --out gpurun_out/r2j_trace.json > gpurun_out/r2j_trace.log 2>&1; tail -2 gpurun_out/r2j_trace.log
timeout 600 python scripts/sweep_opts.py "" "chunk=4" "cluster_route=0" "chunk=4,cluster_route=0" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_c3.py -q -x --timeout 400 -p no:cacheprovider 2>&1 | tail -3
