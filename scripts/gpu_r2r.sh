#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/sweep_opts.py "" "decode_poll_ns=0" "decode_poll_ns=20" "chunk=6" "chunk=12" "tail_per_cta=0" "tail_per_cta=2" "combine_poll_ns=100" 2>&1 | tail -1
touch paper_2502_08246_b200/csrc/decode.cu; make -C paper_2502_08246_b200 NVFLAGS_EXTRA=-DSAAP_REC_RING=6 > /dev/null 2>&1
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
