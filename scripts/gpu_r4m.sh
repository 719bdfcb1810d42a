#!/bin/bash
timeout 240 python scripts/check_tc.py 2>&1 | tail -6
timeout 300 python scripts/sweep_opts.py "" "decode_tc=1" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given "debug_skip=2" "debug_skip=2,decode_tc=1" "decode_tc=1" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "decode_tc=1" "debug_skip=2,decode_tc=1" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --given --opt decode_tc=1 --out gpurun_out/r4n_tc.json > gpurun_out/r4n_a.log 2>&1; tail -c 100 gpurun_out/r4n_a.log
