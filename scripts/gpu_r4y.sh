#!/bin/bash
timeout 600 python scripts/sweep_opts.py "" "guided_div=3" "guided_div=4" "guided_div=3,min_chunk=3" "guided_div=4,min_chunk=2" "guided_div=1" "guided_div=3,claim_lead=4,fetch_lead=3" "chunk=6,guided_div=3" 2>&1 | tail -1
timeout 600 python scripts/sweep_opts.py --given "" "guided_div=3" "guided_div=4" 2>&1 | tail -1
