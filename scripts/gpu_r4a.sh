#!/bin/bash
# late claims (claim_lead / fetch_lead): parity, sweep, tile trace
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_c3.py 2>&1 | tail -3
timeout 900 python scripts/sweep_opts.py "" "claim_lead=8,fetch_lead=8" "claim_lead=2,fetch_lead=1" "claim_lead=4,fetch_lead=2" "claim_lead=3,fetch_lead=1" \
   "min_chunk=2" "min_chunk=1" "min_chunk=2,claim_lead=4" "min_chunk=3" "chunk=6" "chunk=12" "chunk=16,min_chunk=2" 2>&1 | tail -14 > gpurun_out/r4a_sweep.log; cat gpurun_out/r4a_sweep.log | tail -1
timeout 600 python scripts/sweep_opts.py --given "" "min_chunk=2" "claim_lead=4,fetch_lead=2" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --dense "" "min_chunk=2" 2>&1 | tail -1
timeout 600 python scripts/trace_step.py --out gpurun_out/r4a_route.json > gpurun_out/r4a_route.log 2>&1; tail -c 600 gpurun_out/r4a_route.log
