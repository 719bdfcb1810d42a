#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "min_chunk=2" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given --probes 0 "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" "min_chunk=4" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/r3d_pytest.log 2>&1; tail -3 gpurun_out/r3d_pytest.log
