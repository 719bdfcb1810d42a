#!/bin/bash
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given "" "debug_skip=2" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "debug_skip=2" 2>&1 | tail -1
