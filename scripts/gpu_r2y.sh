#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given "" "debug_skip=1" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" 2>&1 | tail -1
