#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "min_chunk=1" "min_chunk=2" 2>&1 | tail -1
timeout 1200 python bench.py --no-imbalanced > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r3f_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['kernel_us'], d['roofline']['frac'], d['parity']['pass'])"; tail -2 gpurun_out/r3f_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/r3f_pytest.log 2>&1; tail -3 gpurun_out/r3f_pytest.log
