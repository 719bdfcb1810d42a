#!/bin/bash
timeout 600 python scripts/sweep_opts.py "" "debug_skip=1" "debug_skip=2" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --given "" "debug_skip=1" "debug_skip=2" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --dense "" "debug_skip=1" "debug_skip=2" 2>&1 | tail -1
