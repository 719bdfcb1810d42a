#!/bin/bash
timeout 150 python scripts/dbg_steps.py --layers 2 --steps 4 2>&1 | tail -4 || exit 1
timeout 900 python scripts/sweep_opts.py "" "claim_lead=8,fetch_lead=8" "claim_lead=2,fetch_lead=1" "claim_lead=4,fetch_lead=2" "claim_lead=3,fetch_lead=1" \
   "min_chunk=2" "min_chunk=1" "min_chunk=2,claim_lead=4" "min_chunk=3" "chunk=6" "chunk=12" "chunk=16,min_chunk=2" 2>&1 | tail -14 > gpurun_out/r4c_sweep.log; cat gpurun_out/r4c_sweep.log | tail -1
