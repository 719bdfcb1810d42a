#!/bin/bash
# diagnose: routed sweep / trace after the late-claim change
mkdir -p gpurun_out
date +%T; timeout 300 python scripts/sweep_opts.py --steps 20 "" 2>&1 | tail -5; date +%T
timeout 200 python scripts/trace_step.py --plain --reps 4 2>&1 | tail -5; date +%T
timeout 200 python scripts/sweep_opts.py --steps 20 "claim_lead=32,fetch_lead=32" 2>&1 | tail -3; date +%T
