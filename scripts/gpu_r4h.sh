#!/bin/bash
timeout 600 python scripts/sweep_opts.py "" "inflight=2" "inflight=1" "combine_poll_ns=200" "combine_poll_ns=0" "combine_poll_ns=3000" "inflight=2,claim_lead=5,fetch_lead=3" "decode_poll_ns=0" "decode_poll_ns=400" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --given "" "inflight=2" "debug_skip=1" "debug_skip=1,inflight=2" "combine_poll_ns=200" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --dense "" "inflight=2" 2>&1 | tail -1
