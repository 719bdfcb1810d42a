#!/bin/bash
timeout 300 python scripts/sweep_opts.py "" "min_chunk=2" "min_chunk=4" "combine_poll_ns=0" "min_chunk=2,combine_poll_ns=0" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense --ctx-len 8192 "" "min_chunk=2" "min_chunk=4" "combine_poll_ns=0" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given --probes 0 "" "combine_poll_ns=0" 2>&1 | tail -1
