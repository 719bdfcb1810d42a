#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --no-imbalanced --no-cpu-baseline > gpurun_out/r3g_bench.json 2> gpurun_out/r3g_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r3g_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['kernel_us'], d['roofline']['frac'])"; tail -2 gpurun_out/r3g_bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_regressions.py tests/test_gpu_cpp_adapter.py -q -x --timeout 400 -p no:cacheprovider 2>&1 | tail -2
