#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/sweep_opts.py "" "chunk=4" "chunk=6" "chunk=3" "chunk=4,tail_per_cta=2" "chunk=4,tail_per_cta=0" "combine_poll_ns=100" "chunk=4,combine_poll_ns=100" "decode_poll_ns=0" "decode_wait=1" 2>&1 | tail -12
